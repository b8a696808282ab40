// Double64 GEMM, bit-exact with the reference.
//
// The reference computes every Double64 output as (kernels.hpp:48-75)
//   acc = 0; for k ascending: acc = fl(acc + fl(a_ik * b_kj));
//   out = fl(alpha * acc); if beta != 0: out = fl(out + fl(beta * c_ij))
// with unfused multiply and add (Release flags, no FMA contraction).  Doing the
// same on the device with __dmul_rn / __dadd_rn -- intrinsics the compiler
// never contracts into DFMA -- in the same k order reproduces its bits, which
// is the reference's own fp64 bar (tests/acceptance.cpp:61-65,
// tests/test_dist_ops.cpp:63-70, 267-306).  Not a tensor-core path: fp64 is
// off the fp32 north star; the kernel is a plain smem-tiled SIMT GEMM.
#include <cuda_runtime.h>

#include <cstdint>

#include "tf32x3_gemm.h"

namespace dm {

namespace {

constexpr int kTile = 64;  // C tile per block (16 x 16 threads, 4 x 4 outputs each)
constexpr int kKT = 16;    // k depth per smem stage

// C[i][j] <- alpha * sum_k A[i][k] B[j][k] (+ beta C[i][j]); A [m x k] and
// B [n x k] K-major (pitches lda, ldb), k strictly ascending per output.
__global__ void __launch_bounds__(256) gemm_f64_exact_kernel(const double* __restrict__ A, int64_t lda,
                                                             const double* __restrict__ B, int64_t ldb, double* C,
                                                             int64_t ldc, int64_t m, int64_t n, int64_t k,
                                                             double alpha, double beta, int read_c) {
  __shared__ double As[kKT][kTile + 1];
  __shared__ double Bs[kKT][kTile + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 16 x 16
  const int t = ty * 16 + tx;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kTile;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kTile;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t k0 = 0; k0 < k; k0 += kKT) {
    // 64 rows x 16 k of each operand: 1024 elements, 4 per thread
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = t + 256 * e;
      const int r = idx / kKT, kk = idx % kKT;
      const int64_t gk = k0 + kk;
      As[kk][r] = (i0 + r < m && gk < k) ? A[(i0 + r) * lda + gk] : 0.0;
      Bs[kk][r] = (j0 + r < n && gk < k) ? B[(j0 + r) * ldb + gk] : 0.0;
    }
    __syncthreads();
    const int kend = static_cast<int>(k - k0 < kKT ? k - k0 : kKT);  // padding must not add +0 terms
    for (int kk = 0; kk < kend; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(av[a], bv[b]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      if (i >= m || j >= n) continue;
      double out = __dmul_rn(alpha, acc[a][b]);
      if (read_c) out = __dadd_rn(out, __dmul_rn(beta, C[i * ldc + j]));
      C[i * ldc + j] = out;
    }
}

// dst[r][k] = trans ? src[k][r] : src[r][k]  (fp64 panel assembly, no rounding)
__global__ void assemble_f64_kernel(const double* __restrict__ src, int64_t lds, int trans, int64_t rows,
                                    int64_t kcols, double* __restrict__ dst, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  if (!trans) {
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int64_t r = r0 + i, kk = k0 + threadIdx.x;
      if (r < rows && kk < kcols) dst[r * ldo + kk] = src[r * lds + kk];
    }
    return;
  }
  for (int i = threadIdx.y; i < 32; i += 8) {  // read src[k][r], coalesced along r
    const int64_t kk = k0 + i, r = r0 + threadIdx.x;
    if (kk < kcols && r < rows) tile[i][threadIdx.x] = src[kk * lds + r];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {  // write dst[r][k], coalesced along k
    const int64_t r = r0 + i, kk = k0 + threadIdx.x;
    if (kk < kcols && r < rows) dst[r * ldo + kk] = tile[threadIdx.x][i];
  }
}

}  // namespace

cudaError_t gemm_f64_exact(const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                           int64_t m, int64_t n, int64_t k, double alpha, double beta, int read_c,
                           cudaStream_t stream) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((n + kTile - 1) / kTile), static_cast<unsigned>((m + kTile - 1) / kTile));
  if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
  gemm_f64_exact_kernel<<<grid, dim3(16, 16), 0, stream>>>(a, lda, b, ldb, c, ldc, m, n, k, alpha, beta, read_c);
  return cudaGetLastError();
}

cudaError_t assemble_f64(const double* src, int64_t lds, int trans, int64_t rows, int64_t kcols, double* dst,
                         int64_t ldo, cudaStream_t stream) {
  if (rows <= 0 || kcols <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((kcols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
  assemble_f64_kernel<<<grid, dim3(32, 8), 0, stream>>>(src, lds, trans, rows, kcols, dst, ldo);
  return cudaGetLastError();
}

}  // namespace dm
