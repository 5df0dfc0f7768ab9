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
// Bump allocator over a pinned host ring, mirrored by a device ring of the
// same size for descriptor lists. Each put records an event (from a reused
// pool); when the ring wraps, every recorded event is waited for, and if the
// device ring was used the device is synchronised as well (a kernel may still
// read descriptors a later copy would overwrite, possibly from another stream).
struct Staging {
    std::mutex mu;
    char* buf = nullptr;    // pinned host ring
    char* dbuf = nullptr;   // device ring (descriptor lists)
    size_t cap = 0, head = 0;
    std::vector<cudaEvent_t> events;
    size_t nev = 0;
    bool dev_used = false;
    static constexpr size_t kMaxEvents = 8192;

    void init() {
        if (buf) return;
        cap = size_t(64) << 20;
        H2B_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf), cap, cudaHostAllocPortable));
    }
    void drain() {
        for (size_t i = 0; i < nev; ++i) H2B_CUDA(cudaEventSynchronize(events[i]));
        if (dev_used) H2B_CUDA(cudaDeviceSynchronize());
        nev = 0;
        head = 0;
        dev_used = false;
    }
    // pinned copy of `host`; returns the ring offset
    size_t reserve(const void* host, size_t bytes) {
        const size_t b = (bytes + 255) & ~size_t(255);
        if (head + b > cap || nev == kMaxEvents) drain();
        const size_t off = head;
        head += b;
        std::memcpy(buf + off, host, bytes);
        return off;
    }
    void record(cudaStream_t s) {
        if (nev == events.size()) {
            cudaEvent_t e;
            H2B_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            events.push_back(e);
        }
        H2B_CUDA(cudaEventRecord(events[nev++], s));
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
        record(s);
        return dst;
    }
    const void* put_dev(const void* host, size_t bytes, cudaStream_t s) {
        std::lock_guard<std::mutex> g(mu);
        if (bytes > (size_t(32) << 20)) return nullptr;
        init();
        if (!dbuf) H2B_CUDA(cudaMalloc(reinterpret_cast<void**>(&dbuf), cap));
        const size_t off = reserve(host, bytes);
        H2B_CUDA(cudaMemcpyAsync(dbuf + off, buf + off, bytes, cudaMemcpyHostToDevice, s));
        record(s);
        dev_used = true;
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

const void* stage_descriptors(const void* host, size_t bytes, cudaStream_t s) {
    return staging().put_dev(host, bytes, s);
}

}  // namespace h2b
