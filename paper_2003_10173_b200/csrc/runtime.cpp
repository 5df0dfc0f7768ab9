// Process-wide device runtime helpers (common.hpp): memory-pool setup and a
// pinned staging ring for host -> device uploads.
#include <cstring>
#include <mutex>
#include <unordered_set>

#include "common.hpp"

namespace h2b {

std::atomic<long long> g_kernel_launches{0};
thread_local bool t_capturing = false;

void ensure_mem_pool() {
    static std::mutex mu;
    static std::unordered_set<int> done;
    int dev = 0;
    H2B_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (done.count(dev)) return;
    cudaMemPool_t pool;
    H2B_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = ~uint64_t(0);
    H2B_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done.insert(dev);
}

namespace {
// Bump allocator over a pinned host ring, mirrored by a device ring of the
// same size for descriptor lists. Puts only copy into the ring and enqueue the
// H2D copy; when the ring wraps, the device is synchronised once (every copy out
// of the ring, and every kernel that may still read a device-ring descriptor
// list, has finished), after which the whole ring is free again. No per-put
// event: HARA issues thousands of small uploads per build.
struct Staging {
    std::mutex mu;
    char* buf = nullptr;    // pinned host ring
    char* dbuf = nullptr;   // device ring (descriptor lists)
    size_t cap = 0, head = 0;
    size_t wraps = 0, puts = 0;

    void init() {
        if (buf) return;
        cap = size_t(64) << 20;
        H2B_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf), cap, cudaHostAllocPortable));
    }
    void drain() {
        H2B_CUDA(cudaDeviceSynchronize());
        head = 0;
        ++wraps;
    }
    // pinned copy of `host`; returns the ring offset
    size_t reserve(const void* host, size_t bytes) {
        const size_t b = (bytes + 255) & ~size_t(255);
        if (head + b > cap) drain();
        const size_t off = head;
        head += b;
        ++puts;
        std::memcpy(buf + off, host, bytes);
        return off;
    }
    void* put(const void* host, size_t bytes, void* dst, cudaStream_t s) {
        std::lock_guard<std::mutex> g(mu);
        if (bytes > (size_t(32) << 20)) {   // huge uploads: plain (synchronising) copy
            H2B_CUDA(cudaMemcpyAsync(dst, host, bytes, cudaMemcpyHostToDevice, s));
            return dst;
        }
        init();
        const size_t off = reserve(host, bytes);
        H2B_CUDA(cudaMemcpyAsync(dst, buf + off, bytes, cudaMemcpyHostToDevice, s));
        return dst;
    }
    const void* put_dev(const void* host, size_t bytes, cudaStream_t s) {
        std::lock_guard<std::mutex> g(mu);
        if (bytes > (size_t(32) << 20)) return nullptr;
        init();
        if (!dbuf) H2B_CUDA(cudaMalloc(reinterpret_cast<void**>(&dbuf), cap));
        const size_t off = reserve(host, bytes);
        H2B_CUDA(cudaMemcpyAsync(dbuf + off, buf + off, bytes, cudaMemcpyHostToDevice, s));
        return dbuf + off;
    }
};
Staging& staging() {
    static Staging* st = new Staging;   // intentionally leaked (lives until process exit)
    return *st;
}
}  // namespace

void* stage_to_device(const void* host, size_t bytes, void* dev_dst, cudaStream_t s) {
    return staging().put(host, bytes, dev_dst, s);
}

void staging_stats(long long* puts, long long* wraps) {
    Staging& st = staging();
    std::lock_guard<std::mutex> g(st.mu);
    if (puts) *puts = static_cast<long long>(st.puts);
    if (wraps) *wraps = static_cast<long long>(st.wraps);
}

const void* stage_descriptors(const void* host, size_t bytes, cudaStream_t s) {
    return staging().put_dev(host, bytes, s);
}

}  // namespace h2b

// diagnostics hook: uploads through the staging ring and ring wraps (device syncs) so far
extern "C" int h2b_staging_stats(long long* puts, long long* wraps) {
    h2b::staging_stats(puts, wraps);
    return 0;
}

// diagnostics hook: kernel launches so far (H2B_LAUNCH sites + replayed graph kernel nodes)
extern "C" long long h2b_kernel_launches(int reset) {
    return reset ? h2b::g_kernel_launches.exchange(0) : h2b::g_kernel_launches.load();
}
