#pragma once
// Error handling and device memory ownership shared by the B200 H^2 library.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <atomic>
#include <stdexcept>
#include <string>
#include <vector>

namespace h2b {

// NVTX range for the duration of a scope (visible in Nsight Systems / ncu
// --nvtx; a few nanoseconds when no tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};


// status codes mirror the reference's exception kinds (include/h2c.h)
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw cuda_error(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " + file + ":" +
                         std::to_string(line));
}
// kernel launches issued so far (diagnostics for bench.py's gpu_launches): every H2B_LAUNCH
// counts one, except while a CUDA graph is being captured; graph replays add their kernel nodes
extern std::atomic<long long> g_kernel_launches;
extern thread_local bool t_capturing;
inline void note_launch(long long k = 1) {
    if (!t_capturing) g_kernel_launches.fetch_add(k, std::memory_order_relaxed);
}
#define H2B_CUDA(x) ::h2b::cuda_check((x), #x, __FILE__, __LINE__)
#define H2B_LAUNCH() (::h2b::note_launch(), ::h2b::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__))

// Device allocations come from the device's stream-ordered memory pool
// (cudaMallocAsync / cudaFreeAsync) with the release threshold raised, so the
// many short-lived H^2 values of a construction recycle HBM without a device
// synchronisation per allocation (cudaMalloc / cudaFree would serialise).
void ensure_mem_pool();

// pinned host staging for small host->device uploads (descriptor lists, plans):
// a pageable cudaMemcpyAsync would synchronise the stream first
void* stage_to_device(const void* host, size_t bytes, void* dev_dst, cudaStream_t s);
// read-only descriptor list for kernels launched on `s`: copied into a device
// ring (no allocation); nullptr when too large for the ring (caller allocates)
const void* stage_descriptors(const void* host, size_t bytes, cudaStream_t s);

// owning device allocation (never host memory); `s` = the stream the buffer is
// allocated on and freed on (nullptr = legacy default stream)
template <class T>
class DeviceArray {
public:
    DeviceArray() = default;
    explicit DeviceArray(size_t n, cudaStream_t s = nullptr) { resize(n, s); }
    ~DeviceArray() { release(); }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    DeviceArray(DeviceArray&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void resize(size_t n, cudaStream_t s = nullptr) {
        if (n == n_) return;
        release();
        s_ = s;
        if (n) {
            ensure_mem_pool();
            H2B_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
        }
        n_ = n;
    }
    void upload(const T* h, size_t n, cudaStream_t s = nullptr) {
        resize(n, s);
        if (n) stage_to_device(h, n * sizeof(T), p_, s);
    }
    void upload(const std::vector<T>& h, cudaStream_t s = nullptr) { upload(h.data(), h.size(), s); }
    std::vector<T> download(cudaStream_t s = nullptr) const {
        std::vector<T> h(n_);
        if (n_) {
            H2B_CUDA(cudaMemcpyAsync(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, s));
            H2B_CUDA(cudaStreamSynchronize(s));
        }
        return h;
    }
    void zero(cudaStream_t s = nullptr) {
        if (n_) H2B_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    T* data() { return p_; }
    const T* data() const { return p_; }
    size_t size() const { return n_; }

private:
    void release() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

}  // namespace h2b
