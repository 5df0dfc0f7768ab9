// Minimal sampling profiler for host code (no perf/gdb in this image).
//   gcc -O2 -shared -fPIC -o tools/sprof.so tools/sprof.c -ldl
//   LD_PRELOAD=tools/sprof.so SPROF_OUT=gpurun_out/sprof.txt python ...
// Every 1 ms of process CPU time (ITIMER_PROF; SPROF_REAL=1: of wall time, ITIMER_REAL) the interrupted thread's stack is
// captured with backtrace(); at exit each sample is written (to $SPROF_OUT.<pid>) as one line of
// "object+offset" frames (innermost first). tools/sprof_report.py symbolizes
// the offsets with addr2line and prints self / inclusive counts per function.
#define _GNU_SOURCE
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/time.h>
#include <unistd.h>

#define MAXS 400000
#define DEPTH 40
static void* g_frames[MAXS][DEPTH];
static int g_depth[MAXS];
static volatile int g_n = 0;
static int g_on = 0;
static int g_real = 0;

static void on_prof(int sig) {
    (void)sig;
    int i = __atomic_fetch_add(&g_n, 1, __ATOMIC_RELAXED);
    if (i >= MAXS) return;
    g_depth[i] = backtrace(g_frames[i], DEPTH);
}

__attribute__((constructor)) static void sprof_init(void) {
    if (!getenv("SPROF_OUT")) return;
    void* warm[4];
    backtrace(warm, 4);   // load the unwinder before the first signal (not async-signal-safe)
    struct sigaction sa;
    memset(&sa, 0, sizeof sa);
    sa.sa_handler = on_prof;
    sa.sa_flags = SA_RESTART;
    // SPROF_REAL=1: sample every 1 ms of WALL time (SIGALRM), so time blocked in
    // synchronisations shows up too; default: every 1 ms of process CPU time
    g_real = getenv("SPROF_REAL") != NULL;
    sigaction(g_real ? SIGALRM : SIGPROF, &sa, NULL);
    struct itimerval it = {{0, 1000}, {0, 1000}};
    setitimer(g_real ? ITIMER_REAL : ITIMER_PROF, &it, NULL);
    g_on = 1;
}

__attribute__((destructor)) static void sprof_fini(void) {
    if (!g_on) return;
    struct itimerval off = {{0, 0}, {0, 0}};
    setitimer(g_real ? ITIMER_REAL : ITIMER_PROF, &off, NULL);
    int n = g_n < MAXS ? g_n : MAXS;
    if (n == 0) return;
    char path[4096];
    snprintf(path, sizeof path, "%s.%d", getenv("SPROF_OUT"), (int)getpid());   // children inherit LD_PRELOAD
    FILE* f = fopen(path, "w");
    if (!f) return;
    for (int i = 0; i < n; ++i) {
        for (int d = 2; d < g_depth[i]; ++d) {   // skip the handler and the signal trampoline
            Dl_info info;
            if (dladdr(g_frames[i][d], &info) && info.dli_fname)
                fprintf(f, "%s+0x%lx ", info.dli_fname,
                        (unsigned long)((char*)g_frames[i][d] - (char*)info.dli_fbase));
            else
                fprintf(f, "?+%p ", g_frames[i][d]);
        }
        fputc('\n', f);
    }
    fclose(f);
}
