// devmem.hpp — minimal device-memory / stream helpers for the host façade.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

namespace gcomm::detail {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw std::runtime_error("no CUDA device: the B200 path has no CPU fallback");
  }
}

// Owning device allocation.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t bytes) { reset(bytes); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
    }
    return *this;
  }
  void reset(std::size_t bytes) {
    release();
    if (bytes) cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc");
    n_ = bytes;
  }
  void ensure(std::size_t bytes) {
    if (bytes > n_) reset(bytes);
  }
  template <class T = void>
  T* get() const { return static_cast<T*>(p_); }
  std::size_t size() const { return n_; }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  void* p_ = nullptr;
  std::size_t n_ = 0;
};

class Stream {
 public:
  Stream() { cuda_check(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "cudaStreamCreate"); }
  ~Stream() { cudaStreamDestroy(s_); }
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
  cudaStream_t get() const { return s_; }
  void sync() const { cuda_check(cudaStreamSynchronize(s_), "cudaStreamSynchronize"); }

 private:
  cudaStream_t s_{};
};

inline std::uint64_t align_up(std::uint64_t x, std::uint64_t a) { return (x + a - 1) / a * a; }

}  // namespace gcomm::detail
