// Host interface of the tcgen05 3xTF32 GEMM (see tf32x3_gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dm {

// C[m x n] (row pitch ldc) <- alpha * A B^T + beta * C, where A and B are
// given as K-major tf32 hi/lo splits: A_{hi,lo} [m x k] pitch lda,
// B_{hi,lo} [n x k] pitch ldb (i.e. op(B) transposed).  read_c == 0 means C
// is never read (reference rule: beta == 0 ignores prior C contents).
struct Tf32x3Args {
  const float* a_hi = nullptr;
  const float* a_lo = nullptr;
  int64_t lda = 0;
  const float* b_hi = nullptr;
  const float* b_lo = nullptr;
  int64_t ldb = 0;
  float* c = nullptr;
  int64_t ldc = 0;
  int64_t m = 0, n = 0, k = 0;
  float alpha = 1.0f, beta = 0.0f;
  int read_c = 0;
  int cta_group = 0;  // 0 = auto, 1 = single-CTA 128x128 tiles, 2 = CTA-pair 256x256 tiles
  int num_sms = 0;    // 0 = all SMs of the current device
  int64_t flush_k = 0;  // K per TMEM accumulation chunk (0 = default 256)
};

cudaError_t tf32x3_gemm(const Tf32x3Args& args, cudaStream_t stream);

// Elementwise split of a strided fp32 panel into K-major tf32 hi/lo planes:
//   out[r][k] = trans ? src[k*lds + r] : src[r*lds + k],  r < rows, k < kcols
// written at hi/lo + r*ldo + k.  `src` may be a peer-GPU (UVA) pointer.
cudaError_t split_tf32(const float* src, int64_t lds, int trans, int64_t rows, int64_t kcols,
                       float* hi, float* lo, int64_t ldo, cudaStream_t stream);

// Seeded synthetic fill, bit-exact with the reference's WorkerContext::fill_seeded
// (runtime_types.hpp:208-218): v[e] = float(2*u53(mix64(key, e)) - 1).
cudaError_t fill_seeded(float* dst, int64_t count, uint64_t key, cudaStream_t stream);

}  // namespace dm
