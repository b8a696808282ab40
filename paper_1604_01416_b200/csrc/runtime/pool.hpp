// Per-worker device memory pool.
//
// Same contract as the reference's host Pool (gridgemm/pool.hpp:22-142):
// power-of-two size classes of at least 64 B, per-class free lists, memory is
// never returned to the driver until trim(), and the Stats record
// {fresh_allocations, reuses, bytes_live, bytes_pooled, high_water}.  On B200
// the point is different -- cudaMalloc/cudaFree synchronise the device and
// IPC-export costs a handle per allocation -- but the observable behaviour
// (a repeated fixed-shape GEMM allocates only on its first iteration,
// tests/acceptance.cpp:437-457) is identical.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.hpp"

namespace dm {

class DevicePool;

// Move-only handle; returns its memory to the owning pool on destruction.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(DeviceBuffer&& o) noexcept { *this = std::move(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      ptr_ = o.ptr_;
      capacity_ = o.capacity_;
      owner_ = o.owner_;
      o.ptr_ = nullptr;
      o.capacity_ = 0;
      o.owner_ = nullptr;
    }
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { reset(); }

  void* data() const { return ptr_; }
  float* f32() const { return static_cast<float*>(ptr_); }
  std::size_t capacity() const { return capacity_; }
  bool valid() const { return ptr_ != nullptr; }
  void reset();

 private:
  friend class DevicePool;
  DeviceBuffer(void* p, std::size_t cap, DevicePool* o) : ptr_(p), capacity_(cap), owner_(o) {}
  void* ptr_ = nullptr;
  std::size_t capacity_ = 0;
  DevicePool* owner_ = nullptr;
};

class DevicePool {
 public:
  struct Stats {
    std::uint64_t fresh_allocations = 0;
    std::uint64_t reuses = 0;
    std::uint64_t bytes_live = 0;
    std::uint64_t bytes_pooled = 0;
    std::uint64_t high_water = 0;
  };
  static constexpr std::size_t kMinClass = 64;

  explicit DevicePool(int device) : device_(device) {}
  DevicePool(const DevicePool&) = delete;
  DevicePool& operator=(const DevicePool&) = delete;
  ~DevicePool() { release_all(); }

  static std::size_t size_class(std::size_t bytes) {
    std::size_t cls = kMinClass;
    while (cls < bytes) cls <<= 1;
    return cls;
  }

  DeviceBuffer acquire(std::size_t bytes) {
    if (bytes == 0) throw UsageError("pool_acquire: zero-byte request");
    std::lock_guard<std::mutex> lk(mu_);
    const std::size_t cls = size_class(bytes);
    auto& list = free_lists_[cls];
    void* p = nullptr;
    if (!list.empty()) {
      p = list.back();
      list.pop_back();
      stats_.reuses += 1;
      stats_.bytes_pooled -= cls;
    } else {
      int prev = -1;
      cudaGetDevice(&prev);
      cudaSetDevice(device_);
      cudaError_t e = cudaMalloc(&p, cls);
      if (e == cudaErrorMemoryAllocation && stats_.bytes_pooled > 0) {
        // out of memory with idle pooled blocks of other classes: return them
        // to the driver and retry once (the reference's host pool would page)
        cudaGetLastError();
        release_pooled_locked();
        e = cudaMalloc(&p, cls);
      }
      if (prev >= 0) cudaSetDevice(prev);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw CudaError("pool_acquire: cudaMalloc of " + std::to_string(cls) + " bytes failed: " +
                        cudaGetErrorString(e));
      }
      stats_.fresh_allocations += 1;
      ++generation_;
    }
    stats_.bytes_live += cls;
    live_[p] = cls;
    const std::uint64_t total = stats_.bytes_live + stats_.bytes_pooled;
    if (total > stats_.high_water) stats_.high_water = total;
    return DeviceBuffer(p, cls, this);
  }

  void release(DeviceBuffer& b) {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = live_.find(b.ptr_);
    if (b.owner_ != this || it == live_.end())
      throw UsageError("pool_release: buffer does not belong to this pool");
    live_.erase(it);
    stats_.bytes_live -= b.capacity_;
    stats_.bytes_pooled += b.capacity_;
    free_lists_[b.capacity_].push_back(b.ptr_);
    b.ptr_ = nullptr;
    b.owner_ = nullptr;
    b.capacity_ = 0;
  }

  // Frees every pooled buffer; live buffers stay live (pool.hpp:110-115).
  std::uint64_t trim() {
    std::lock_guard<std::mutex> lk(mu_);
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    const std::uint64_t freed = release_pooled_locked();
    if (prev >= 0) cudaSetDevice(prev);
    return freed;
  }

  // (mu_ held, device_ current) free every idle pooled block
  std::uint64_t release_pooled_locked() {
    const std::uint64_t freed = stats_.bytes_pooled;
    for (auto& [cls, list] : free_lists_)
      for (void* p : list) cudaFree(p);
    free_lists_.clear();
    stats_.bytes_pooled = 0;
    ++generation_;
    return freed;
  }

  Stats stats() const {
    std::lock_guard<std::mutex> lk(mu_);
    return stats_;
  }
  int device() const { return device_; }
  // Bumped whenever the set of driver allocations changes (IPC re-export).
  std::uint64_t generation() const { return generation_; }

 private:
  void release_all() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    for (auto& [cls, list] : free_lists_)
      for (void* p : list) cudaFree(p);
    for (auto& [p, cls] : live_) cudaFree(p);
    if (prev >= 0) cudaSetDevice(prev);
    free_lists_.clear();
    live_.clear();
  }

  int device_;
  mutable std::mutex mu_;
  std::map<std::size_t, std::vector<void*>> free_lists_;
  std::unordered_map<void*, std::size_t> live_;
  Stats stats_;
  std::uint64_t generation_ = 0;
};

inline void DeviceBuffer::reset() {
  if (ptr_ != nullptr && owner_ != nullptr) owner_->release(*this);
}

}  // namespace dm
