// Error taxonomy, hashing and seed mixing of the distributed-matrix runtime.
//
// Mirrors the reference's error classes (gridgemm/common.hpp:22-78) so every
// C-ABI status code maps 1:1 onto the exception a reference user expects, and
// restates its FNV-1a (common.hpp:83-103) and splitmix64 seed mixer
// (common.hpp:107-121) -- the latter defines the seeded synthetic inputs.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../../include/dmath_b200.h"

namespace dm {

// Current-device scope (restores the caller's device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Integer tuning knob from the environment (read per call, so tests and
// benches can flip schedules between commands).
inline std::int64_t env_int(const char* name, std::int64_t dflt) {
  const char* v = std::getenv(name);
  if (v == nullptr || *v == 0) return dflt;
  return std::strtoll(v, nullptr, 10);
}

// Host-side phase timer (DM_HOST_PROF=1): accumulated wall time per named
// phase of the command path, printed to stderr at exit.  Diagnostic only.
struct HostProf {
  struct Acc {
    double us = 0;
    long n = 0;
  };
  std::map<std::string, Acc> acc;
  std::mutex mu;
  static HostProf& get() {
    static HostProf* p = new HostProf();  // leaked on purpose: printed from atexit
    return *p;
  }
  static bool on() {
    static const bool v = env_int("DM_HOST_PROF", 0) != 0;
    return v;
  }
  ~HostProf() = default;
};
inline void host_prof_dump() {
  HostProf& h = HostProf::get();
  std::lock_guard<std::mutex> lk(h.mu);
  for (const auto& [k, a] : h.acc)
    std::fprintf(stderr, "[host-prof] %-28s %10.2f us/call  (%ld calls)\n", k.c_str(), a.us / std::max(1L, a.n), a.n);
}
struct HostScope {
  const char* name;
  std::chrono::steady_clock::time_point t0;
  explicit HostScope(const char* n) : name(n) {
    if (HostProf::on()) t0 = std::chrono::steady_clock::now();
  }
  ~HostScope() {
    if (!HostProf::on()) return;
    const double us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    HostProf& h = HostProf::get();
    static bool registered = [] { return std::atexit(host_prof_dump) == 0; }();
    (void)registered;
    std::lock_guard<std::mutex> lk(h.mu);
    auto& a = h.acc[name];
    a.us += us;
    a.n += 1;
  }
};

// DM_GEMM_MODE environment default of the split-product scheme (0 = 3xTF32,
// 1 = mixed, 3 = f16x2, anything else / unset = auto), as kernel mode
// constants (kModeTf32x3 = 0, kModeMixed = 1, kModeAuto = 2, kModeF16x2 = 3).
inline int env_gemm_mode() {
  const std::int64_t v = env_int("DM_GEMM_MODE", 2);
  return v == 0 ? 0 : v == 1 ? 1 : v == 3 ? 3 : 2;
}

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

#define DM_DEFINE_ERROR(Name, Code) \
  class Name : public Error {       \
   public:                          \
    explicit Name(const std::string& w) : Error(Code, w) {} \
  };

DM_DEFINE_ERROR(UsageError, DM_ERR_USAGE)
DM_DEFINE_ERROR(ConfigError, DM_ERR_CONFIG)
DM_DEFINE_ERROR(ShapeError, DM_ERR_SHAPE)
DM_DEFINE_ERROR(ProtocolError, DM_ERR_PROTOCOL)
DM_DEFINE_ERROR(PlanError, DM_ERR_PLAN)
DM_DEFINE_ERROR(IntegrityError, DM_ERR_INTEGRITY)
DM_DEFINE_ERROR(UnsupportedError, DM_ERR_UNSUPPORTED)
DM_DEFINE_ERROR(CudaError, DM_ERR_CUDA)
DM_DEFINE_ERROR(NcclError, DM_ERR_NCCL)
#undef DM_DEFINE_ERROR

class CacheMissError : public Error {
 public:
  CacheMissError(const std::string& w, std::vector<std::pair<int, int>> missing)
      : Error(DM_ERR_CACHE_MISS, w), missing_coords(std::move(missing)) {}
  std::vector<std::pair<int, int>> missing_coords;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                    ")");
}

inline DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev);
  cuda_check(cudaSetDevice(dev), "cudaSetDevice");
}

// FNV-1a 64 (descriptor digests; checksums of gathered matrices in tests).
class Fnv1a {
 public:
  void update(const void* data, std::size_t n) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < n; ++i) {
      state_ ^= p[i];
      state_ *= 1099511628211ULL;
    }
  }
  void update_u64(std::uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    update(b, 8);
  }
  std::uint64_t digest() const { return state_; }

 private:
  std::uint64_t state_ = 14695981039346656037ULL;
};

inline std::uint64_t mix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b) { return mix64(a ^ mix64(b)); }

}  // namespace dm
