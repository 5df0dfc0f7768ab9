#pragma once
// Error handling and device memory ownership shared by the B200 H^2 library.
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace h2b {

// status codes mirror the reference's exception kinds (include/h2c.h)
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw cuda_error(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " + file + ":" +
                         std::to_string(line));
}
#define H2B_CUDA(x) ::h2b::cuda_check((x), #x, __FILE__, __LINE__)
#define H2B_LAUNCH() ::h2b::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// owning device allocation (cudaMalloc; never host memory)
template <class T>
class DeviceArray {
public:
    DeviceArray() = default;
    explicit DeviceArray(size_t n) { resize(n); }
    ~DeviceArray() { release(); }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    DeviceArray(DeviceArray&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void resize(size_t n) {
        if (n == n_) return;
        release();
        if (n) H2B_CUDA(cudaMalloc(&p_, n * sizeof(T)));
        n_ = n;
    }
    void upload(const T* h, size_t n, cudaStream_t s = 0) {
        resize(n);
        if (n) H2B_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& h, cudaStream_t s = 0) { upload(h.data(), h.size(), s); }
    std::vector<T> download(cudaStream_t s = 0) const {
        std::vector<T> h(n_);
        if (n_) {
            H2B_CUDA(cudaMemcpyAsync(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, s));
            H2B_CUDA(cudaStreamSynchronize(s));
        }
        return h;
    }
    void zero(cudaStream_t s = 0) {
        if (n_) H2B_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    T* data() { return p_; }
    const T* data() const { return p_; }
    size_t size() const { return n_; }

private:
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* p_ = nullptr;
    size_t n_ = 0;
};

}  // namespace h2b
