// Data operations beside the GEMM; see dataops.h.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dataops.h"

namespace dm {

namespace {

// ---- scalar rules of the reference: widen exactly, narrow once (RNE) ----
template <int P> struct Scalar;
template <> struct Scalar<0> { using T = __half; using Acc = float; };
template <> struct Scalar<1> { using T = float; using Acc = float; };
template <> struct Scalar<2> { using T = double; using Acc = double; };

template <int P>
__device__ __forceinline__ double to_double(const typename Scalar<P>::T* p) {
  if constexpr (P == 0) return static_cast<double>(__half2float(*p));
  else return static_cast<double>(*p);
}

template <int P>
__device__ __forceinline__ typename Scalar<P>::Acc to_acc(const typename Scalar<P>::T* p) {
  if constexpr (P == 0) return __half2float(*p);
  else return *p;
}

// scalar_from_double (precision.hpp:83-89) for each storage precision.
template <int P>
__device__ __forceinline__ void from_double(double v, typename Scalar<P>::T* out) {
  if constexpr (P == 2) {
    *out = v;
  } else if constexpr (P == 1) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    if ((b & 0x7FF0000000000000ull) == 0x7FF0000000000000ull && (b & 0xFFFFFFFFFFFFFull)) {
      // NaN: quiet, payload truncated to the top fraction bits (static_cast<float>)
      const unsigned s = static_cast<unsigned>(b >> 63) << 31;
      *out = __uint_as_float(s | 0x7FC00000u | static_cast<unsigned>((b >> 29) & 0x7FFFFFull));
    } else {
      *out = __double2float_rn(v);
    }
  } else {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    if ((b & 0x7FF0000000000000ull) == 0x7FF0000000000000ull && (b & 0xFFFFFFFFFFFFFull)) {
      // NaN: keep the top payload bits, never collapse to inf (half.hpp:19-25)
      unsigned short pay = static_cast<unsigned short>((b >> 42) & 0x3FFull);
      if (pay == 0) pay = 0x200;
      const unsigned short s = static_cast<unsigned short>((b >> 48) & 0x8000ull);
      *out = __ushort_as_half(static_cast<unsigned short>(s | 0x7C00u | pay));
    } else {
      *out = __double2half(v);  // round to nearest even
    }
  }
}

template <int P>
__device__ __forceinline__ void from_acc(typename Scalar<P>::Acc v, typename Scalar<P>::T* out) {
  from_double<P>(static_cast<double>(v), out);
}

template <int SP, int DP>
__global__ void convert_kernel(const void* src, void* dst, int64_t count) {
  const auto* s = static_cast<const typename Scalar<SP>::T*>(src);
  auto* d = static_cast<typename Scalar<DP>::T*>(dst);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    from_double<DP>(to_double<SP>(s + i), d + i);
}

template <int SP, int DP>
__global__ void remap_kernel(const void* const* src_blocks, void* dst, RemapGeometry g) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i >= g.dst_rows || j >= g.dst_cols) return;
  const int64_t lin = (g.r0 + i) * g.dst_gcols + (g.c0 + j);
  const int64_t sr = lin / g.src_gcols, sc = lin - sr * g.src_gcols;
  const int64_t br = sr / g.src_brows, bc = sc / g.src_bcols;
  const int64_t bcols = min(g.src_bcols, g.src_gcols - bc * g.src_bcols);  // trimmed edge block
  const auto* blk = static_cast<const typename Scalar<SP>::T*>(src_blocks[br * g.src_nbc + bc]);
  const typename Scalar<SP>::T* p = blk + (sr - br * g.src_brows) * bcols + (sc - bc * g.src_bcols);
  auto* d = static_cast<typename Scalar<DP>::T*>(dst);
  from_double<DP>(to_double<SP>(p), d + i * g.dst_cols + j);
}

template <int P>
__global__ void partial_kernel(const void* const* blocks, const int64_t* inner, const int64_t* pitch,
                               int nlanes, int axis, int64_t len, void* out) {
  using T = typename Scalar<P>::T;
  using Acc = typename Scalar<P>::Acc;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    Acc acc = Acc(0);
    for (int l = 0; l < nlanes; ++l) {
      const T* b = static_cast<const T*>(blocks[l]);
      const int64_t n = inner[l], ld = pitch[l];
      if (axis == 0) {
        const T* row = b + i * ld;
        for (int64_t k = 0; k < n; ++k) acc = acc + to_acc<P>(row + k);
      } else {
        for (int64_t k = 0; k < n; ++k) acc = acc + to_acc<P>(b + k * ld + i);
      }
    }
    from_acc<P>(acc, static_cast<T*>(out) + i);
  }
}

template <int P>
__global__ void fold_kernel(const void* const* parts, int nparts, int64_t len, void* out) {
  using T = typename Scalar<P>::T;
  using Acc = typename Scalar<P>::Acc;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    Acc acc = Acc(0);
    for (int p = 0; p < nparts; ++p) acc = acc + to_acc<P>(static_cast<const T*>(parts[p]) + i);
    from_acc<P>(acc, static_cast<T*>(out) + i);
  }
}

unsigned blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t convert_copy(const void* src, int sp, void* dst, int dp, int64_t count,
                         cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  if (sp == dp) return cudaMemcpyAsync(dst, src, count * precision_bytes(sp), cudaMemcpyDefault, stream);
  const unsigned g = blocks_for(count, 256);
#define DM_CONV(S, D) \
  if (sp == S && dp == D) convert_kernel<S, D><<<g, 256, 0, stream>>>(src, dst, count);
  DM_CONV(0, 1) DM_CONV(0, 2) DM_CONV(1, 0) DM_CONV(1, 2) DM_CONV(2, 0) DM_CONV(2, 1)
#undef DM_CONV
  return cudaGetLastError();
}

cudaError_t remap_gather(const void* const* src_blocks, int sp, void* dst, int dp,
                         const RemapGeometry& geo, cudaStream_t stream) {
  if (geo.dst_rows <= 0 || geo.dst_cols <= 0) return cudaSuccess;
  dim3 block(32, 8);
  dim3 grid(static_cast<unsigned>((geo.dst_cols + 31) / 32), static_cast<unsigned>((geo.dst_rows + 7) / 8));
  if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
#define DM_REMAP(S, D) \
  if (sp == S && dp == D) remap_kernel<S, D><<<grid, block, 0, stream>>>(src_blocks, dst, geo);
  DM_REMAP(0, 0) DM_REMAP(0, 1) DM_REMAP(0, 2) DM_REMAP(1, 0) DM_REMAP(1, 1) DM_REMAP(1, 2)
  DM_REMAP(2, 0) DM_REMAP(2, 1) DM_REMAP(2, 2)
#undef DM_REMAP
  return cudaGetLastError();
}

cudaError_t segment_partial(const void* const* blocks, const int64_t* inner, const int64_t* pitch,
                            int nlanes, int axis, int prec, int64_t len, void* out,
                            cudaStream_t stream) {
  if (len <= 0) return cudaSuccess;
  const unsigned g = blocks_for(len, 128);
  if (prec == 0) partial_kernel<0><<<g, 128, 0, stream>>>(blocks, inner, pitch, nlanes, axis, len, out);
  else if (prec == 1) partial_kernel<1><<<g, 128, 0, stream>>>(blocks, inner, pitch, nlanes, axis, len, out);
  else partial_kernel<2><<<g, 128, 0, stream>>>(blocks, inner, pitch, nlanes, axis, len, out);
  return cudaGetLastError();
}

cudaError_t fold_partials(const void* const* parts, int nparts, int prec, int64_t len, void* out,
                          cudaStream_t stream) {
  if (len <= 0) return cudaSuccess;
  const unsigned g = blocks_for(len, 256);
  if (prec == 0) fold_kernel<0><<<g, 256, 0, stream>>>(parts, nparts, len, out);
  else if (prec == 1) fold_kernel<1><<<g, 256, 0, stream>>>(parts, nparts, len, out);
  else fold_kernel<2><<<g, 256, 0, stream>>>(parts, nparts, len, out);
  return cudaGetLastError();
}

}  // namespace dm
