// Process-wide device runtime helpers (common.hpp): memory-pool setup and a
// pinned staging ring for host -> device uploads.
#include <cstring>
#include <mutex>
#include <unordered_set>

#include "common.hpp"

namespace h2b {

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
// bump allocator over a pinned buffer; when full, wait for every stream that
// copied out of it (events) and start over
struct Staging {
    std::mutex mu;
    char* buf = nullptr;
    size_t cap = 0, head = 0;
    std::vector<cudaEvent_t> pending;
    ~Staging() {
        // process teardown: the driver reclaims pinned memory and events
    }
    void* put(const void* host, size_t bytes, void* dst, cudaStream_t s) {
        std::lock_guard<std::mutex> g(mu);
        if (bytes > (size_t(32) << 20)) {   // huge uploads: plain (synchronising) copy
            H2B_CUDA(cudaMemcpyAsync(dst, host, bytes, cudaMemcpyHostToDevice, s));
            return dst;
        }
        if (!buf) {
            cap = size_t(64) << 20;
            H2B_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf), cap, cudaHostAllocPortable));
        }
        const size_t b = (bytes + 255) & ~size_t(255);
        if (head + b > cap) {
            for (cudaEvent_t e : pending) {
                H2B_CUDA(cudaEventSynchronize(e));
                cudaEventDestroy(e);
            }
            pending.clear();
            head = 0;
        }
        char* p = buf + head;
        head += b;
        std::memcpy(p, host, bytes);
        H2B_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s));
        cudaEvent_t e;
        H2B_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        H2B_CUDA(cudaEventRecord(e, s));
        pending.push_back(e);
        if (pending.size() > 4096) {   // bound the event list
            for (cudaEvent_t x : pending) {
                H2B_CUDA(cudaEventSynchronize(x));
                cudaEventDestroy(x);
            }
            pending.clear();
            head = 0;
        }
        return dst;
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

}  // namespace h2b
