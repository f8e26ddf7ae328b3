// device_utils.cuh — CUDA error checking and a minimal owning device buffer.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>
#include <vector>

#include "common.hpp"

namespace hfmm_b200 {

#define HFMM_CUDA_CHECK(expr)                                                              \
  do {                                                                                     \
    cudaError_t err__ = (expr);                                                            \
    if (err__ != cudaSuccess)                                                              \
      throw ::hfmm_b200::Error(HFMM_ERR_DEVICE, std::string(#expr) + ": " +                \
                                                    cudaGetErrorString(err__));            \
  } while (0)

// bytes currently held through DeviceBuffer on this process (reported in hfmm_cuda_stats)
size_t& device_bytes_counter();

template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) { resize(n); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(o.ptr_), n_(o.n_) { o.ptr_ = nullptr; o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      ptr_ = o.ptr_;
      n_ = o.n_;
      o.ptr_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DeviceBuffer() { release(); }

  void resize(size_t n) {
    if (n == n_) return;
    release();
    if (n) {
      HFMM_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&ptr_), n * sizeof(T)));
      device_bytes_counter() += n * sizeof(T);
    }
    n_ = n;
  }
  void release() {
    if (ptr_) {
      cudaFree(ptr_);
      device_bytes_counter() -= n_ * sizeof(T);
    }
    ptr_ = nullptr;
    n_ = 0;
  }
  void upload(const T* host, size_t n, cudaStream_t s = 0) {
    resize(n);
    if (n) HFMM_CUDA_CHECK(cudaMemcpyAsync(ptr_, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s = 0) { upload(v.data(), v.size(), s); }
  void download(T* host, size_t n, cudaStream_t s = 0) const {
    if (n) HFMM_CUDA_CHECK(cudaMemcpyAsync(host, ptr_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void zero(cudaStream_t s = 0) {
    if (n_) HFMM_CUDA_CHECK(cudaMemsetAsync(ptr_, 0, n_ * sizeof(T), s));
  }
  T* get() const { return ptr_; }
  size_t size() const { return n_; }

 private:
  T* ptr_ = nullptr;
  size_t n_ = 0;
};

}  // namespace hfmm_b200
