// Data-movement kernels that feed the 3xTF32 GEMM.
//
// split_tf32: reads a (possibly transposed, possibly peer-GPU) fp32 panel and
//   writes the K-major tf32 hi/lo planes consumed by tf32x3_gemm.  This replaces
//   the reference's panel assembly `assemble_op_rows` / `assemble_op_cols`
//   (/root/reference/proj/include/gridgemm/ops.hpp:177-208, 534-558), fused with
//   the 3xTF32 split; when `src` is a peer pointer it is also the transfer.
// fill_seeded: bit-exact device restatement of WorkerContext::fill_seeded
//   (runtime_types.hpp:208-218) using mix64 / u64_to_unit_double
//   (common.hpp:107-121).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "split_common.cuh"
#include "tf32x3_gemm.h"

namespace dm {

namespace {

using splitdev::Planes;
using splitdev::split_store;
using splitdev::split_store4;

constexpr int kT = 32;  // tile edge
constexpr int kRowsPerPass = 8;

template <typename T>
__device__ __forceinline__ float load_widen(const T* p) {
  if constexpr (sizeof(T) == 2) return __half2float(__ldg(reinterpret_cast<const __half*>(p)));
  else return __ldg(p);
}

// One 32x32 output tile per block (32 x 8 threads).
template <typename T>
__global__ void split_direct_kernel(const T* __restrict__ src, int64_t lds, int64_t rows,
                                    int64_t kcols, Planes p) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kT;
  if (k >= kcols) return;
#pragma unroll
  for (int i = 0; i < kT; i += kRowsPerPass) {
    const int64_t r = r0 + threadIdx.y + i;
    if (r < rows) split_store(load_widen(src + r * lds + k), p, r, k, splitdev::row_exp(p, r));
  }
}

template <typename T>
__global__ void split_trans_kernel(const T* __restrict__ src, int64_t lds, int64_t rows,
                                   int64_t kcols, Planes p) {
  __shared__ float tile[kT][kT + 1];
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * kT;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kT;
  // read: src[k][r], coalesced along r
#pragma unroll
  for (int i = 0; i < kT; i += kRowsPerPass) {
    const int64_t k = k0 + threadIdx.y + i, r = r0 + threadIdx.x;
    if (k < kcols && r < rows) tile[threadIdx.y + i][threadIdx.x] = load_widen(src + k * lds + r);
  }
  __syncthreads();
  // write: out[r][k], coalesced along k
#pragma unroll
  for (int i = 0; i < kT; i += kRowsPerPass) {
    const int64_t r = r0 + threadIdx.y + i, k = k0 + threadIdx.x;
    if (k < kcols && r < rows) split_store(tile[threadIdx.x][threadIdx.y + i], p, r, k, splitdev::row_exp(p, r));
  }
}

// ---- vectorised fp32 variants: 4 consecutive elements per access, 4 accesses
// in flight per thread.
// (4*WY) rows x 128 k per block (32 x WY threads); requires 16-B aligned rows.
// (Measured 6.6 TB/s of HBM traffic at 1 GiB input; later K panels are split
// by the GEMM's own split warps instead, see tf32x3_gemm.cu.)
template <int WY>
__global__ void __launch_bounds__(32 * WY, 48 / WY) split_direct_vec4_kernel(const float* __restrict__ src,
                                                                            int64_t lds, int64_t rows,
                                                                            int64_t kcols, Planes p) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * 128 + threadIdx.x * 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * (4 * WY);
  if (k >= kcols) return;
  float4 v[4];
  const bool full = k + 4 <= kcols;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + threadIdx.y + WY * i;
    if (r < rows && full) v[i] = __ldg(reinterpret_cast<const float4*>(src + r * lds + k));
  }
  int e[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + threadIdx.y + WY * i;
    e[i] = r < rows ? splitdev::row_exp(p, r) : 0;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + threadIdx.y + WY * i;
    if (r >= rows) continue;
    if (full) {
      split_store4(v[i], p, r, k, e[i]);
    } else {
      for (int64_t kk = k; kk < kcols; ++kk) split_store(__ldg(src + r * lds + kk), p, r, kk, e[i]);
    }
  }
}

// out[r][k] = src[k][r]: 64 k x 128 r per block through shared memory.
// Reads: 512-B row segments, all of a thread's float4 loads in flight before
// the smem stores.  Writes: a thread pair per output row, the pair's float4s
// interleaved by 4 k (conflict-free smem reads), 32 B sectors complete.
constexpr int kTransK = 64;
template <int WY>
__global__ void __launch_bounds__(32 * WY, 24 / WY) split_trans_vec4_kernel(const float* __restrict__ src,
                                                                           int64_t lds, int64_t rows,
                                                                           int64_t kcols, Planes p) {
  __shared__ __align__(16) float tile[kTransK][128 + 4];
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * kTransK;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 128;
  const int t = threadIdx.y * 32 + threadIdx.x;
  const int64_t r = r0 + threadIdx.x * 4;
  constexpr int kLoads = kTransK / WY;
  constexpr int kBatch = kLoads < 8 ? kLoads : 8;
  const bool full_r = r + 4 <= rows;
#pragma unroll
  for (int i0 = 0; i0 < kLoads; i0 += kBatch) {
    float4 v[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t k = k0 + threadIdx.y + WY * (i0 + i);
      if (k < kcols && full_r) v[i] = __ldcs(reinterpret_cast<const float4*>(src + k * lds + r));
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int kl = threadIdx.y + WY * (i0 + i);
      if (k0 + kl >= kcols) continue;
      if (full_r) {
        *reinterpret_cast<float4*>(&tile[kl][threadIdx.x * 4]) = v[i];
      } else {
        for (int u = 0; u < 4; ++u)
          if (r + u < rows) tile[kl][threadIdx.x * 4 + u] = __ldcs(src + (k0 + kl) * lds + r + u);
      }
    }
  }
  __syncthreads();
  for (int rl = t >> 1; rl < 128; rl += 16 * WY) {
    const int64_t ro = r0 + rl;
    if (ro >= rows) break;
    const int e = splitdev::row_exp(p, ro);
#pragma unroll
    for (int j = 0; j < kTransK / 8; ++j) {
      const int kl = 8 * j + 4 * (t & 1);
      const int64_t k = k0 + kl;
      if (k >= kcols) continue;
      if (k + 4 <= kcols) {
        split_store4(make_float4(tile[kl][rl], tile[kl + 1][rl], tile[kl + 2][rl], tile[kl + 3][rl]), p,
                     ro, k, e);
      } else {
        for (int u = 0; k + u < kcols; ++u) split_store(tile[kl + u][rl], p, ro, k + u, e);
      }
    }
  }
}

// f16x2 planes from a direct source (op(X) rows stored as rows): each
// thread splits 8 consecutive k of 4 rows -- two float4 loads per row, all
// eight in flight -- and stores 16 B of h0 and of h1 per row, so a warp store
// covers 512 contiguous bytes of a plane row; 32 rows x 256 k per block.
__global__ void __launch_bounds__(256, 4) split_direct_f16x2_kernel(const float* __restrict__ src, int64_t lds,
                                                                    int64_t rows, int64_t kcols, Planes p) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t k = static_cast<int64_t>(blockIdx.x) * 256 + tx * 8;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32 + ty;
  if (k >= kcols) return;
  const bool full = k + 8 <= kcols;
  float4 v[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + 8 * i;
    if (r < rows && full) {
      const float4* q = reinterpret_cast<const float4*>(src + r * lds + k);
      v[i][0] = __ldcs(q);
      v[i][1] = __ldcs(q + 1);
    }
  }
  int e[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + 8 * i;
    e[i] = r < rows ? splitdev::row_exp(p, r) : 0;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + 8 * i;
    if (r >= rows) break;
    if (full) {
      const float x[8] = {v[i][0].x, v[i][0].y, v[i][0].z, v[i][0].w, v[i][1].x, v[i][1].y, v[i][1].z, v[i][1].w};
      uint32_t h[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = splitdev::scale_pow2(x[2 * u], e[i]), b = splitdev::scale_pow2(x[2 * u + 1], e[i]);
        __half2 hh = __floats2half2_rn(a, b);
        const float2 hf = __half22float2(hh);
        __half2 ll = __floats2half2_rn(a - hf.x, b - hf.y);
        h[u] = *reinterpret_cast<uint32_t*>(&hh);
        l[u] = *reinterpret_cast<uint32_t*>(&ll);
      }
      __stcs(reinterpret_cast<uint4*>(p.h0 + r * p.ldo16 + k), make_uint4(h[0], h[1], h[2], h[3]));
      __stcs(reinterpret_cast<uint4*>(p.h1 + r * p.ldo16 + k), make_uint4(l[0], l[1], l[2], l[3]));
    } else {
      for (int64_t kk = k; kk < kcols; ++kk) splitdev::split_store(__ldcs(src + r * lds + kk), p, r, kk, e[i]);
    }
  }
}

// f16x2 planes from a transposed source, out[r][k] = src[k][r] (the op(B)^T
// rows of a non-transposed B): 64 k x 128 r per block through a 32 KB smem
// tile whose 16-B column groups are XOR-swizzled by k / 8.  The write phase
// gives each output row 8 threads of 8 consecutive k (16 B of h0 and of h1
// per thread), so one warp store fills four 128-B row segments -- where the
// tf32-shaped kernel above writes 16 rows x 16 B per store -- and its smem
// reads (8 k of one r per thread) hit 32 distinct banks.
__global__ void __launch_bounds__(256, 4) split_trans_f16x2_kernel(const float* __restrict__ src, int64_t lds,
                                                                   int64_t rows, int64_t kcols, Planes p) {
  __shared__ __align__(16) float tile[64][128];
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 128;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r = r0 + tx * 4;
  // load: warp ty takes k rows ty, ty + 8, ..., all eight float4 in flight
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t k = k0 + ty + 8 * i;
    v[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (k < kcols) {
      if (r + 4 <= rows) {
        v[i] = __ldcs(reinterpret_cast<const float4*>(src + k * lds + r));
      } else {
        float* f = reinterpret_cast<float*>(&v[i]);
        for (int u = 0; u < 4; ++u)
          if (r + u < rows) f[u] = __ldcs(src + k * lds + r + u);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)  // row kl = ty + 8 i, column group tx ^ i (kl >> 3 == i)
    *reinterpret_cast<float4*>(&tile[ty + 8 * i][4 * (tx ^ i)]) = v[i];
  __syncthreads();
  // write: lane = 4 c + s -> k chunk c (8 k), row s of a group of four rows
  const int c = tx >> 2, s = tx & 3;
  const int64_t kk = k0 + 8 * c;
  if (kk >= kcols) return;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    const int rl = 4 * (8 * pass + ty) + s;
    const int64_t ro = r0 + rl;
    if (ro >= rows) break;
    const int e = splitdev::row_exp(p, ro);
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = tile[8 * c + u][rl ^ (4 * c)];
    if (kk + 8 <= kcols) {
      uint32_t h[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = splitdev::scale_pow2(x[2 * u], e), b = splitdev::scale_pow2(x[2 * u + 1], e);
        __half2 hh = __floats2half2_rn(a, b);
        const float2 hf = __half22float2(hh);
        __half2 ll = __floats2half2_rn(a - hf.x, b - hf.y);
        h[u] = *reinterpret_cast<uint32_t*>(&hh);
        l[u] = *reinterpret_cast<uint32_t*>(&ll);
      }
      __stcs(reinterpret_cast<uint4*>(p.h0 + ro * p.ldo16 + kk), make_uint4(h[0], h[1], h[2], h[3]));
      __stcs(reinterpret_cast<uint4*>(p.h1 + ro * p.ldo16 + kk), make_uint4(l[0], l[1], l[2], l[3]));
    } else {
      for (int u = 0; kk + u < kcols; ++u) splitdev::split_store(x[u], p, ro, kk + u, e);
    }
  }
}

template <int WY>
void launch_split_vec4(const float* s32, int64_t lds, int trans, int64_t rows, int64_t kcols, const Planes& p,
                       cudaStream_t stream) {
  const dim3 block(32, WY);
  if (trans) {
    const dim3 g(static_cast<unsigned>((kcols + kTransK - 1) / kTransK), static_cast<unsigned>((rows + 127) / 128));
    split_trans_vec4_kernel<WY><<<g, block, 0, stream>>>(s32, lds, rows, kcols, p);
  } else {
    const dim3 g(static_cast<unsigned>((kcols + 127) / 128), static_cast<unsigned>((rows + 4 * WY - 1) / (4 * WY)));
    split_direct_vec4_kernel<WY><<<g, block, 0, stream>>>(s32, lds, rows, kcols, p);
  }
}

int split_warps() {
  static const int w = [] {
    const char* e = std::getenv("DM_SPLIT_WARPS");
    const int v = e ? std::atoi(e) : 8;
    return (v == 2 || v == 4) ? v : 8;
  }();
  return w;
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

template <typename T>
__global__ void fill_seeded_kernel(T* __restrict__ dst, int64_t count, uint64_t key) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = mix64(key ^ mix64(static_cast<uint64_t>(e)));
    const double u = static_cast<double>(h >> 11) * 0x1.0p-53;
    const double v = 2.0 * u - 1.0;
    if constexpr (sizeof(T) == 8) dst[e] = v;
    else if constexpr (sizeof(T) == 4) dst[e] = __double2float_rn(v);
    else dst[e] = __double2half(v);  // RNE from double, as half_bits_from_double
  }
}

// ---- per-row |x| maxima for the scaled 2xFP16 split (kModeF16x2)
// rmax[r] = max(rmax[r], max_k |x[r][k]|) as float bits (non-negative floats
// order like their bits, so atomicMax on unsigned is a float max).
// Direct: one warp per row and 4096-k slice, float4 loads when aligned.
__global__ void __launch_bounds__(256) absmax_direct_kernel(const float* __restrict__ src, int64_t lds,
                                                            int64_t rows, int64_t kcols, unsigned* rmax) {
  const int64_t r = static_cast<int64_t>(blockIdx.y) * 8 + threadIdx.x / 32;
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 4096;
  const int64_t k1 = min(kcols, k0 + 4096);
  const float* row = src + r * lds;
  float m = 0.0f;
  int64_t kv = k0;
  if ((reinterpret_cast<uintptr_t>(row + k0) & 15) == 0) {
    for (; kv + 128 <= k1; kv += 128) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(row + kv) + lane);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
  for (int64_t k = kv + lane; k < k1; k += 32) m = fmaxf(m, fabsf(__ldcs(row + k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0 && m > 0.0f) atomicMax(rmax + r, __float_as_uint(m));
}

// Transposed (x[r][k] = src[k * lds + r]): 128 rows x 256 k per block, each
// thread 4 adjacent r (float4 along the contiguous axis) over 32 k.
__global__ void __launch_bounds__(256) absmax_trans_kernel(const float* __restrict__ src, int64_t lds,
                                                           int64_t rows, int64_t kcols, unsigned* rmax) {
  __shared__ float red[8][128];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r = static_cast<int64_t>(blockIdx.y) * 128 + tx * 4;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 256;
  const bool vec = r + 4 <= rows && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (lds & 3) == 0;
  float m[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int i = 0; i < 32; ++i) {
    const int64_t k = k0 + ty + 8 * i;
    if (k >= kcols) break;
    if (vec) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(src + k * lds + r));
      m[0] = fmaxf(m[0], fabsf(v.x));
      m[1] = fmaxf(m[1], fabsf(v.y));
      m[2] = fmaxf(m[2], fabsf(v.z));
      m[3] = fmaxf(m[3], fabsf(v.w));
    } else {
      for (int u = 0; u < 4; ++u)
        if (r + u < rows) m[u] = fmaxf(m[u], fabsf(__ldcs(src + k * lds + r + u)));
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) red[ty][tx * 4 + u] = m[u];
  __syncthreads();
  if (threadIdx.x < 128) {
    float v = red[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 8; ++y) v = fmaxf(v, red[y][threadIdx.x]);
    const int64_t rr = static_cast<int64_t>(blockIdx.y) * 128 + threadIdx.x;
    if (rr < rows && v > 0.0f) atomicMax(rmax + rr, __float_as_uint(v));
  }
}

// dst[r] = max over the n sources of src[i][r] (row maxima as float bits;
// sources may live on peer GPUs).
__global__ void rowmax_combine_kernel(RowmaxSources srcs, unsigned* __restrict__ dst, int64_t rows) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    unsigned m = 0;
    for (int i = 0; i < srcs.n; ++i) m = max(m, __ldcg(srcs.p[i] + r));
    dst[r] = m;
  }
}

}  // namespace

cudaError_t rowmax_combine(const RowmaxSources& srcs, unsigned* dst, int64_t rows, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (srcs.n < 1 || srcs.n > RowmaxSources::kMax) return cudaErrorInvalidValue;
  const int blocks = static_cast<int>(std::min<int64_t>((rows + 255) / 256, 148 * 4));
  rowmax_combine_kernel<<<blocks, 256, 0, stream>>>(srcs, dst, rows);
  return cudaGetLastError();
}

cudaError_t split_tf32(const void* src, int src_half, int64_t lds, int trans, int64_t rows,
                       int64_t kcols, float* hi, float* lo, int64_t ldo, void* hi16, void* lo16,
                       int64_t ldo16, cudaStream_t stream) {
  if (rows <= 0 || kcols <= 0) return cudaSuccess;
  Planes p{hi, lo, static_cast<__nv_bfloat16*>(hi16), static_cast<__nv_bfloat16*>(lo16), ldo, ldo16};
  dim3 block(kT, kRowsPerPass);
  dim3 grid(static_cast<unsigned>((kcols + kT - 1) / kT), static_cast<unsigned>((rows + kT - 1) / kT));
  if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
  if (src_half) {
    const __half* s16 = static_cast<const __half*>(src);
    if (trans) split_trans_kernel<<<grid, block, 0, stream>>>(s16, lds, rows, kcols, p);
    else split_direct_kernel<<<grid, block, 0, stream>>>(s16, lds, rows, kcols, p);
  } else {
    const float* s32 = static_cast<const float*>(src);
    auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    auto a8 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 7) == 0; };
    // vector path: 16-B aligned source rows and destination rows
    const bool vec = a16(s32) && (lds & 3) == 0 && a16(hi) && (ldo & 3) == 0 &&
                     (lo == nullptr || a16(lo)) &&
                     (hi16 == nullptr || (a8(hi16) && a8(lo16) && (ldo16 & 3) == 0));
    if (vec) {
      if ((rows + 7) / 8 > 65535) return cudaErrorInvalidConfiguration;
      switch (split_warps()) {
        case 2: launch_split_vec4<2>(s32, lds, trans, rows, kcols, p, stream); break;
        case 4: launch_split_vec4<4>(s32, lds, trans, rows, kcols, p, stream); break;
        default: launch_split_vec4<8>(s32, lds, trans, rows, kcols, p, stream); break;
      }
      return cudaGetLastError();
    }
    if (trans) split_trans_kernel<<<grid, block, 0, stream>>>(s32, lds, rows, kcols, p);
    else split_direct_kernel<<<grid, block, 0, stream>>>(s32, lds, rows, kcols, p);
  }
  return cudaGetLastError();
}

cudaError_t absmax_rows(const float* src, int64_t lds, int trans, int64_t rows, int64_t kcols, unsigned* rmax,
                        cudaStream_t stream) {
  if (rows <= 0 || kcols <= 0) return cudaSuccess;
  if (trans) {
    const dim3 g(static_cast<unsigned>((kcols + 255) / 256), static_cast<unsigned>((rows + 127) / 128));
    if (g.y > 65535u) return cudaErrorInvalidConfiguration;
    absmax_trans_kernel<<<g, 256, 0, stream>>>(src, lds, rows, kcols, rmax);
  } else {
    const dim3 g(static_cast<unsigned>((kcols + 4095) / 4096), static_cast<unsigned>((rows + 7) / 8));
    if (g.y > 65535u) return cudaErrorInvalidConfiguration;
    absmax_direct_kernel<<<g, 256, 0, stream>>>(src, lds, rows, kcols, rmax);
  }
  return cudaGetLastError();
}

cudaError_t split_f16x2(const float* src, int64_t lds, int trans, int64_t rows, int64_t kcols, void* h0, void* h1,
                        int64_t ldo16, const unsigned* rmax, cudaStream_t stream) {
  if (rows <= 0 || kcols <= 0) return cudaSuccess;
  Planes p{nullptr, nullptr, nullptr, nullptr, 0, ldo16};
  p.h0 = static_cast<__half*>(h0);
  p.h1 = static_cast<__half*>(h1);
  p.rmax = rmax;
  auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  auto a8 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 7) == 0; };
  const char* t16 = std::getenv("DM_SPLIT_TRANS16");  // 0: the tf32-shaped transposing kernel (A/B, tests)
  const bool trans16 = t16 == nullptr || std::atoi(t16) != 0;
  const char* d16 = std::getenv("DM_SPLIT_DIRECT16");  // 0: the tf32-shaped direct kernel (A/B, tests)
  const bool direct16 = d16 == nullptr || std::atoi(d16) != 0;
  if (!trans && direct16 && a16(src) && (lds & 3) == 0 && a16(h0) && a16(h1) && (ldo16 & 7) == 0) {
    const dim3 g(static_cast<unsigned>((kcols + 255) / 256), static_cast<unsigned>((rows + 31) / 32));
    if (g.y > 65535u) return cudaErrorInvalidConfiguration;
    split_direct_f16x2_kernel<<<g, 256, 0, stream>>>(src, lds, rows, kcols, p);
    return cudaGetLastError();
  }
  if (trans && trans16 && a16(src) && (lds & 3) == 0 && a16(h0) && a16(h1) && (ldo16 & 7) == 0) {
    const dim3 g(static_cast<unsigned>((kcols + 63) / 64), static_cast<unsigned>((rows + 127) / 128));
    if (g.y > 65535u) return cudaErrorInvalidConfiguration;
    split_trans_f16x2_kernel<<<g, 256, 0, stream>>>(src, lds, rows, kcols, p);
    return cudaGetLastError();
  }
  if (a16(src) && (lds & 3) == 0 && a8(h0) && a8(h1) && (ldo16 & 3) == 0) {
    if ((rows + 7) / 8 > 65535) return cudaErrorInvalidConfiguration;
    switch (split_warps()) {
      case 2: launch_split_vec4<2>(src, lds, trans, rows, kcols, p, stream); break;
      case 4: launch_split_vec4<4>(src, lds, trans, rows, kcols, p, stream); break;
      default: launch_split_vec4<8>(src, lds, trans, rows, kcols, p, stream); break;
    }
    return cudaGetLastError();
  }
  dim3 block(kT, kRowsPerPass);
  dim3 grid(static_cast<unsigned>((kcols + kT - 1) / kT), static_cast<unsigned>((rows + kT - 1) / kT));
  if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
  if (trans) split_trans_kernel<<<grid, block, 0, stream>>>(src, lds, rows, kcols, p);
  else split_direct_kernel<<<grid, block, 0, stream>>>(src, lds, rows, kcols, p);
  return cudaGetLastError();
}

cudaError_t fill_seeded(void* dst, int precision, int64_t count, uint64_t key, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  const unsigned g = static_cast<unsigned>(blocks);
  if (precision == 0) fill_seeded_kernel<<<g, 256, 0, stream>>>(static_cast<__half*>(dst), count, key);
  else if (precision == 2) fill_seeded_kernel<<<g, 256, 0, stream>>>(static_cast<double*>(dst), count, key);
  else fill_seeded_kernel<<<g, 256, 0, stream>>>(static_cast<float*>(dst), count, key);
  return cudaGetLastError();
}

}  // namespace dm
