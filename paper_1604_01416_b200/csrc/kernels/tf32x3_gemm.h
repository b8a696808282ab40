// Host interface of the tcgen05 3xTF32 GEMM (see tf32x3_gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

namespace dm {

// Split-product modes.  All keep fp32 accuracy:
//   kModeTf32x3 : acc += lo*hi + hi*lo + hi*hi, three kind::tf32 MMAs per k8 step
//   kModeMixed  : acc += hi*hi (kind::tf32) + bf16(hi)*bf16(lo) + bf16(lo)*bf16(hi)
//                 (kind::f16, bf16 inputs): the cross terms are 2^-11 smaller than
//                 the product and need only bf16's 8 bits; BF16 MMAs run at twice
//                 the TF32 rate, so a k16 step costs 4 TF32-MMA slots instead of 6.
constexpr int kModeTf32x3 = 0;
constexpr int kModeMixed = 1;
constexpr int kModeAuto = 2;
//   kModeF16x2  : scaled 2xFP16 -- per plane row x 2^e = h0 + h1 with fp16 h0, h1
//                 (11 + 11 bits, the precision of 3xTF32's tf32 hi / lo pair),
//                 acc += h1*h0 + h0*h1 + h0*h0, three kind::f16 MMAs per k16
//                 (3 slots vs mixed's 4 and 3xTF32's 6); the epilogue undoes the
//                 power-of-two scales (split_common.cuh).  4 B of planes per element.
constexpr int kModeF16x2 = 3;
// kModeAuto runs every fp32 product in kModeF16x2: measured on B200
// (tools/f16x2_probe.py, profiles/r02/f16x2/) it has 3xTF32's accuracy -- the
// same 11 + 11-bit pair and three products; within 1.0-1.5x of 3xTF32's
// distance from the exact product over U[-1,1), U[0,1), log-uniform 2^+-20 and
// 2^+-60, rows spanning 2^+-60, K = 256 .. 32768 -- at 1.8x its speed
// (N=32768: 462 vs 260 TFLOP/s; mixed: 310, with a bf16 floor of ~6e-7).
// Except for latency-bound products: below DM_F16X2_MIN_GFLOP (default 64)
// of work, auto runs 3xTF32, whose one-pass split beats f16x2's row-maxima
// pass + split where the GEMM itself takes microseconds (BASELINE config 1,
// 2048^3 on 4 GPUs: f16x2 splits 95 us vs the batched 3xTF32 split's 27 us).
// `work` = 2 m n k of the launch / worker (< 0: unknown, treated as large).
inline int resolve_split_mode(int mode, int64_t /*k_total*/, double work = -1.0) {
  if (mode != kModeAuto) return mode;
  if (work >= 0.0) {
    const char* v = std::getenv("DM_F16X2_MIN_GFLOP");
    const double min_gflop = (v != nullptr && *v != 0) ? std::strtod(v, nullptr) : 64.0;
    if (work < min_gflop * 1e9) return kModeTf32x3;
  }
  return kModeF16x2;
}

// One split job fused into a GEMM launch: the split_tf32 of an fp32 piece
// (16-B aligned rows and planes) for the NEXT K panel, executed by the
// kernel's two split warps while its tensor-core pipeline runs.  With `flag`
// set, the job's source is a landing buffer filled by copy-engine transfers:
// the warps wait until (int)(*flag - flag_val) >= 0 before reading it.
struct SplitJob {
  const float* src = nullptr;
  unsigned* rmax = nullptr;  // kModeF16x2: row maxima of the target planes (hi16 / lo16 = fp16 h0 / h1)
  int64_t lds = 0;
  int trans = 0;
  int64_t rows = 0, kcols = 0;
  float* hi = nullptr;
  float* lo = nullptr;
  void* hi16 = nullptr;
  void* lo16 = nullptr;
  int64_t ldo = 0, ldo16 = 0;
  const unsigned* flag = nullptr;
  unsigned flag_val = 0;
  int64_t t0 = 0;  // first tile of this job in the launch's concatenated tile space
};
constexpr int kMaxSplitJobs = 16;
struct SplitJobs {
  SplitJob job[kMaxSplitJobs];
  int n = 0;
  // kModeF16x2 jobs run in two phases (row maxima, then the split) with a
  // grid-wide handoff on this zeroed counter (fused: every CTA of the GEMM
  // launch arrives once; requires the launch's CTAs to be co-resident)
  unsigned* phase_ctr = nullptr;
  int64_t t_begin = 0, t_end = 0;  // tile range this launch processes
};
// tiles of one job (direct: 32 rows x 128 k; transposed: 32 k x 128 rows)
int64_t split_job_tiles(const SplitJob& j);
// can the GEMM's split warps run this job (fp32, aligned)?
bool split_job_fusable(const SplitJob& j);
// Run a list of split jobs (no landing flags, all fusable) as one kernel
// launch over their concatenated tiles [t_begin, t_end).
cudaError_t split_jobs(const SplitJobs& jobs, cudaStream_t stream);

// C[m x n] (row pitch ldc) <- alpha * A B^T + beta * C, where A and B are
// given as split planes, each either K-major -- A [m x k], B [n x k] (i.e.
// op(B) transposed), fp32 containers pitch lda/ldb, bf16 planes lda16/ldb16 --
// or MN-major (a_mn / b_mn): A [k x m], B [k x n] with the pitches along m / n
// (a multiple of 4 fp32 / 8 bf16 elements).  MN-major lets a transposed
// operand be split without a transpose.
// read_c == 0 means C is never read (reference rule: beta == 0 ignores C).
struct Tf32x3Args {
  const float* a_hi = nullptr;   // tf32-rounded hi (fp32 container)
  const float* a_lo = nullptr;   // kModeTf32x3: tf32 lo
  const void* a_hi16 = nullptr;  // kModeMixed: bf16(hi)
  const void* a_lo16 = nullptr;  // kModeMixed: bf16(lo)
  int64_t lda = 0, lda16 = 0;
  const float* b_hi = nullptr;
  const float* b_lo = nullptr;
  const void* b_hi16 = nullptr;
  const void* b_lo16 = nullptr;
  int64_t ldb = 0, ldb16 = 0;
  const unsigned* a_max = nullptr;  // kModeF16x2: row maxima of op(A) / op(B)^T planes (a/b_hi16 = h0,
  const unsigned* b_max = nullptr;  // a/b_lo16 = h1, fp16, K-major)
  int mode = kModeTf32x3;
  int a_mn = 0, b_mn = 0;  // planes MN-major instead of K-major
  int a_mn16 = -1, b_mn16 = -1;  // bf16 planes' majorness when it differs (-1: as a_mn / b_mn)
  float* c = nullptr;   // fp32 C, or fp16 C (reinterpreted) when c_half != 0
  int c_half = 0;       // Half16 storage: beta*C widened exactly, result rounded RNE once
  int64_t ldc = 0;
  int64_t m = 0, n = 0, k = 0;
  float alpha = 1.0f, beta = 0.0f;
  int read_c = 0;
  int cta_group = 0;  // 0 = auto, 1 = single-CTA 128x128 tiles, 2 = CTA-pair 256x256 tiles
  int num_sms = 0;    // 0 = all SMs of the current device
  int64_t flush_k = 0;  // K per TMEM accumulation chunk (0 = tf32x3_default_flush_k)
  int64_t k_total = 0;  // K of the whole product when this launch is one K panel of it (0 = k)
  int group_m = 0;      // rasterisation group of m-tiles (0 = default)
  int l2_policy = 1;    // TMA L2 hint: 0 evict_normal, 1 evict_last, 2 evict_first
  int lockstep = 0;     // >0: producers stay within this many k-blocks of each other
  unsigned* sync = nullptr;  // lockstep counters (>= tf32x3_sync_bytes), private to this launch
  size_t sync_bytes = 0;
  const SplitJobs* split = nullptr;  // fused split work for this launch (may be null)
  int ksplit = 0;         // split-K: 0 auto (tiles cannot fill the SMs), 1 off, >1 forced
  float* ws = nullptr;    // split-K partials (>= tf32x3_splitk_bytes); no workspace = no split
  size_t ws_bytes = 0;
  int c_prefetch = -1;    // beta != 0: L2 prefetch of C this many TMEM chunks ahead (0 / -1: off; measured no gain)
};

cudaError_t tf32x3_gemm(const Tf32x3Args& args, cudaStream_t stream);

// Default TMEM accumulation chunk for a product over k_total.  The tensor
// core adds each MMA into its fp32 accumulator with truncation, so a chunk's
// error grows with the MMAs issued into it; chunks are folded into an fp32
// register master with round-to-nearest adds.  Shorter chunks cost epilogue
// time (measured at 16384^3, mixed: 256 -> 280, 128 -> 269, 64 -> 260
// TFLOP/s), so they are used where the reference's own k-ascending fp32 loop
// is most accurate (small K): the chunk keeps the split GEMM's error at or
// below the reference's at every K (profiles/r02/flush_probe.log).
int64_t tf32x3_default_flush_k(int mode, int64_t k_total);

// Bytes of lockstep counters a launch with these arguments needs (0 if off).
// Lockstep requires every CTA of the launch to be co-resident: do not enable it
// when other persistent kernels can share the device concurrently.
size_t tf32x3_sync_bytes(const Tf32x3Args& args);

// Workspace bytes for the split-K partials this launch would use (0: none).
size_t tf32x3_splitk_bytes(const Tf32x3Args& args);

// Elementwise split of a strided fp32 panel into K-major planes:
//   x[r][k] = trans ? src[k*lds + r] : src[r*lds + k],  r < rows, k < kcols
//   hi = rn_tf32(x) at hi + r*ldo + k;   lo = x - hi rounded to tf32 (lo != null)
//   and/or bf16(hi), bf16(lo) at hi16/lo16 + r*ldo16 + k (when non-null).
// `src` may be a peer-GPU (UVA / IPC-mapped) pointer: the pull and the split are
// one kernel.
// `src_half` != 0: the source holds fp16 scalars, widened exactly (the
// reference's AccumOf<Half> = float, kernels.hpp:29-35).
cudaError_t split_tf32(const void* src, int src_half, int64_t lds, int trans, int64_t rows,
                       int64_t kcols, float* hi, float* lo, int64_t ldo, void* hi16, void* lo16,
                       int64_t ldo16, cudaStream_t stream);

// kModeF16x2 planes.  absmax_rows: rmax[r] = max(rmax[r], max_k |x[r][k]|) as
// float bits, x as in split_tf32 (rmax zeroed by the caller before the first
// piece of a plane).  split_f16x2: h0 / h1 fp16 planes (pitch ldo16) of x[r][k]
// scaled by 2^e(rmax[r]) (split_common.cuh).
cudaError_t absmax_rows(const float* src, int64_t lds, int trans, int64_t rows, int64_t kcols, unsigned* rmax,
                        cudaStream_t stream);
cudaError_t split_f16x2(const float* src, int64_t lds, int trans, int64_t rows, int64_t kcols, void* h0, void* h1,
                        int64_t ldo16, const unsigned* rmax, cudaStream_t stream);
// Row maxima of a whole op(X) row from its blocks' partial maxima:
// dst[r] = max_i p[i][r] (float bits; p[i] may point into peer memory).
struct RowmaxSources {
  static constexpr int kMax = 32;
  const unsigned* p[kMax];
  int n = 0;
};
cudaError_t rowmax_combine(const RowmaxSources& srcs, unsigned* dst, int64_t rows, cudaStream_t stream);

// Double64 GEMM bit-exact with the reference's gemm_typed<double> (gemm_f64.cu):
// C[i][j] <- alpha * sum_k A[i][k] B[j][k] (+ beta C[i][j] when read_c), A and B
// K-major, k ascending, unfused multiply and add.
cudaError_t gemm_f64_exact(const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                           int64_t m, int64_t n, int64_t k, double alpha, double beta, int read_c,
                           cudaStream_t stream);
// fp64 panel assembly: dst[r][k] = trans ? src[k*lds + r] : src[r*lds + k].
cudaError_t assemble_f64(const double* src, int64_t lds, int trans, int64_t rows, int64_t kcols, double* dst,
                         int64_t ldo, cudaStream_t stream);

// Stream-ordered 32-bit store without an SM (a stream memory operation):
// *addr = value once the stream's earlier work (e.g. copy-engine transfers)
// completed; pairs with SplitJob::flag.
cudaError_t stream_write_flag(cudaStream_t stream, unsigned* addr, unsigned value);

// Seeded synthetic fill, bit-exact with the reference's WorkerContext::fill_seeded
// (runtime_types.hpp:208-218): v[e] = T(2*u53(mix64(key, e)) - 1), the double
// narrowed once with round-to-nearest-even (scalar_from_double, precision.hpp:83-89).
// precision: 0 Half16, 1 Single32, 2 Double64.
cudaError_t fill_seeded(void* dst, int precision, int64_t count, uint64_t key, cudaStream_t stream);

}  // namespace dm
