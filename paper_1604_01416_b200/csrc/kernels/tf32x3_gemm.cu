// 3xTF32 fp32-accurate GEMM on the sm_100a 5th-generation tensor cores.
//
// This is the B200 replacement for the reference's per-worker BLAS seam
// `gridgemm::local_gemm` -> `detail::gemm_typed<float>`
// (/root/reference/proj/include/gridgemm/kernels.hpp:48-89):
//
//     C <- alpha * op(A) op(B) + beta * C      (beta == 0 never reads C)
//
// Operands arrive pre-split (split_pack.cu) as K-major tf32 hi/lo pairs:
//     x = hi + lo,  hi = rn_tf32(x),  lo = rn_tf32(x - hi)
// and the product is accumulated in fp32 TMEM as
//     acc += lo_A*hi_B + hi_A*lo_B + hi_A*hi_B      (lo*lo dropped, ~2^-22)
//
// Structure (one persistent CTA per SM, or one CTA pair per TPC for CG=2):
//   warp 0      TMA producer   4 tiles per stage (A hi/lo, B hi/lo), 128B swizzle
//   warp 1      MMA issuer     tcgen05.mma.kind::tf32, 3 MMAs per k8 step; owns TMEM
//   warps 2..9  epilogue       tcgen05.ld -> fp32 master (RN) -> alpha/beta -> stores
// Pipelines: smem full/empty mbarriers (TMA<->MMA) and double-buffered TMEM
// K-chunk accumulators with full/empty mbarriers (MMA<->epilogue).
//
// CG=1: tile 128x128 (UMMA M=128,N=128), cta_group::1.
// CG=2: CTA pair computes a 256x256 tile (UMMA M=256,N=256, cta_group::2);
//       each CTA stages its 128 rows of A and 128 rows of B^T, the leader
//       issues the MMAs, both CTAs drain their own 128 accumulator lanes.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <atomic>
#include <cstdio>

#include "../runtime/common.hpp"
#include "ptx.cuh"
#include "split_common.cuh"
#include "tf32x3_gemm.h"

namespace dm {

namespace {

template <int CG>
struct Cfg {
  static constexpr int kRowsPerCta = 128;              // A rows and B rows staged per CTA
  static constexpr int kUmmaM = 128 * CG;
  static constexpr int kUmmaN = 128 * CG;
  static constexpr int kBK = 32;                       // fp32 per 128-B swizzle row
  static constexpr int kStages = 3;
  static constexpr int kTileBytes = kRowsPerCta * kBK * 4;  // 16 KB
  static constexpr int kStageBytes = 4 * kTileBytes;        // 64 KB
  static constexpr int kAccCols = kUmmaN;                    // fp32 TMEM columns per chunk buffer
  static constexpr int kTmemCols = 2 * kAccCols;             // double-buffered chunks
  static constexpr int kEpiWarps = 8;                        // 2 per TMEM lane quadrant
  static constexpr int kColsPerThread = kAccCols / 2;        // master accumulator registers
  static constexpr int kSplitWarps = 2;                      // fused split of the next panel
  static constexpr int kThreads = 64 + 32 * kEpiWarps + 32 * kSplitWarps;
  static constexpr int kSplitTileBytes = 32 * (128 + 4) * 4;  // transposed split tile
  static constexpr int kSmemBytes =
      kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/ + kSplitTileBytes;
};

struct EpiParams {
  float* c;
  int c_half;
  int64_t ldc;
  int m, n;
  float alpha, beta;
  int read_c;
  int group_m;          // rasterisation: tiles walk n inside groups of group_m m-tiles
  int l2_policy;        // 0 evict_normal, 1 evict_last, 2 evict_first (TMA cache hint)
  int lockstep;         // >0: producers of a wave stay within `lockstep` k-blocks
  unsigned* sync;       // lockstep counters [waves * epochs], zeroed per launch
  int ksplit;           // >1: split-K; item (s, tile) writes its fp32 partial to ws[s]
  float* ws;            // [ksplit][m][n] partial tiles (ksplit > 1)
  int a_mn, b_mn;       // fp32 operand planes MN-major (M / N contiguous) instead of K-major
  int a_mn16, b_mn16;   // the same for the bf16 planes (mixed mode)
  const unsigned* a_max;  // kModeF16x2: row maxima of the A / B^T planes (power-of-two scales)
  const unsigned* b_max;
  int c_prefetch;         // beta != 0: prefetch the tile's C rows into L2 this many chunks before its end (0 off)
};

// k per pipeline stage: 32 fp32 or 64 fp16 elements fill a 128-B swizzle row
template <int MODE>
__host__ __device__ constexpr int stage_k() { return MODE == kModeF16x2 ? 64 : 32; }

// Work item t of a launch: tile t % tiles of K-split t / tiles, whose k-blocks
// are [kb_lo, kb_hi) (empty ranges still store a zero partial).
__device__ __forceinline__ void item_range(int t, int total_tiles, int num_kb, int ksplit, int& tile, int& split,
                                           int& kb_lo, int& kb_hi) {
  split = t / total_tiles;
  tile = t - split * total_tiles;
  const int per = (num_kb + ksplit - 1) / ksplit;
  kb_lo = min(num_kb, split * per);
  kb_hi = min(num_kb, kb_lo + per);
}

template <int CG>
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int G, int& mt, int& nt) {
  const int per_group = G * tiles_n;
  const int group = t / per_group;
  const int first_m = group * G;
  const int gsize = min(G, tiles_m - first_m);
  const int r = t - group * per_group;
  mt = first_m + r % gsize;
  nt = r / gsize;
}

// ---------------------------------------------------------------- split warps
// The kernel's two split warps run split jobs for the next K panel (see
// SplitJob) while the producer / MMA / epilogue warps run this panel: the
// split then needs no SM time of its own (a separate split kernel cannot be
// co-resident with this one -- the GEMM's warps leave too few registers in
// every SM sub-partition), and no launch between the panels' GEMMs.
// Tiles: direct 32 rows x 128 k (16 float4 loads in flight per thread),
// transposed 32 k x 128 rows through a shared-memory tile.
__device__ __forceinline__ void split_bar() { asm volatile("bar.sync 1, 64;" ::: "memory"); }

// Job j of tile t, waiting for its landing flag the first time (`ready` bits).
__device__ __forceinline__ const SplitJob& split_job_of(const SplitJobs& sj, int64_t t, uint32_t& ready) {
  int j = 0;
  while (j + 1 < sj.n && t >= sj.job[j + 1].t0) ++j;
  const SplitJob& jb = sj.job[j];
  if (jb.flag != nullptr && !(ready & (1u << j))) {
    const long long t0 = clock64();
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(jb.flag) : "memory");
      if (static_cast<int>(v - jb.flag_val) >= 0) break;
      __nanosleep(256);
      if (clock64() - t0 > (1ll << 36)) __trap();  // landing copy never signalled
    }
    ready |= 1u << j;
  }
  return jb;
}

// Phase 1 of kModeF16x2 jobs: per plane row, the |x| maximum of this block's
// tiles into jb.rmax (atomicMax on the float bits).  Same tiles as the split.
__device__ __noinline__ void run_absmax_jobs(const SplitJobs& sj, int st, uint32_t& ready) {
  const int lane = st & 31, wy = st >> 5;
  for (int64_t t = sj.t_begin + blockIdx.x; t < sj.t_end; t += gridDim.x) {
    const SplitJob& jb = split_job_of(sj, t, ready);
    const int64_t lt = t - jb.t0;
    if (!jb.trans) {
      const int64_t tiles_k = (jb.kcols + 127) / 128;
      const int64_t k = (lt % tiles_k) * 128 + lane * 4;
      const int64_t r0 = (lt / tiles_k) * 32 + wy;
      // all 16 rows' loads in flight before any reduction (a peer source
      // costs an NVLink round trip per dependent load)
      float m[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t r = r0 + 2 * i;
        m[i] = 0.0f;
        if (r < jb.rows && k + 4 <= jb.kcols) {
          const float4 v = __ldcs(reinterpret_cast<const float4*>(jb.src + r * jb.lds + k));
          m[i] = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
        } else if (r < jb.rows) {
          for (int64_t kk = k; kk < jb.kcols; ++kk) m[i] = fmaxf(m[i], fabsf(__ldcs(jb.src + r * jb.lds + kk)));
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t r = r0 + 2 * i;
        if (r >= jb.rows) break;  // warp-uniform
        float mi = m[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mi = fmaxf(mi, __shfl_xor_sync(0xffffffffu, mi, o));
        if (lane == 0 && mi > 0.0f) atomicMax(jb.rmax + r, __float_as_uint(mi));
      }
    } else {
      const int64_t tiles_k = (jb.kcols + 31) / 32;
      const int64_t k0 = (lt % tiles_k) * 32;
      const int64_t r = (lt / tiles_k) * 128 + lane * 4;
      float m[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t k = k0 + wy + 2 * i;
        if (k >= jb.kcols) continue;
        if (r + 4 <= jb.rows) {
          const float4 v = __ldcs(reinterpret_cast<const float4*>(jb.src + k * jb.lds + r));
          m[0] = fmaxf(m[0], fabsf(v.x));
          m[1] = fmaxf(m[1], fabsf(v.y));
          m[2] = fmaxf(m[2], fabsf(v.z));
          m[3] = fmaxf(m[3], fabsf(v.w));
        } else {
          for (int u = 0; u < 4; ++u)
            if (r + u < jb.rows) m[u] = fmaxf(m[u], fabsf(__ldcs(jb.src + k * jb.lds + r + u)));
        }
      }
      for (int u = 0; u < 4; ++u)
        if (r + u < jb.rows && m[u] > 0.0f) atomicMax(jb.rmax + r + u, __float_as_uint(m[u]));
    }
  }
}

// phase: 0 split only; 1 row maxima only (kModeF16x2, separate launch);
// 2 both, with a grid-wide handoff on sj.phase_ctr in between (fused into a
// persistent GEMM launch, whose CTAs are all co-resident).
__device__ __noinline__ void run_split_jobs(const SplitJobs& sj, float (*tile)[128 + 4], int st, int phase) {
  using splitdev::Planes;
  const int lane = st & 31, wy = st >> 5;
  uint32_t ready = 0;  // jobs whose landing flag was seen
  if (phase != 0) {
    run_absmax_jobs(sj, st, ready);
    if (phase == 1) return;
    split_bar();
    if (st == 0) {
      __threadfence();
      atomicAdd(sj.phase_ctr, 1u);
      const long long t0 = clock64();
      while (true) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sj.phase_ctr) : "memory");
        if (v >= gridDim.x) break;
        __nanosleep(128);
        if (clock64() - t0 > (1ll << 36)) __trap();  // a CTA of the launch never arrived
      }
    }
    split_bar();
  }
  for (int64_t t = sj.t_begin + blockIdx.x; t < sj.t_end; t += gridDim.x) {
    const SplitJob& jb = split_job_of(sj, t, ready);
    Planes p{jb.hi, jb.lo, static_cast<__nv_bfloat16*>(jb.hi16), static_cast<__nv_bfloat16*>(jb.lo16),
             jb.ldo, jb.ldo16};
    if (jb.rmax != nullptr) {
      p = Planes{nullptr, nullptr, nullptr, nullptr, 0, jb.ldo16};
      p.h0 = static_cast<__half*>(jb.hi16);
      p.h1 = static_cast<__half*>(jb.lo16);
      p.rmax = jb.rmax;
    }
    const int64_t lt = t - jb.t0;
    if (!jb.trans) {
      const int64_t tiles_k = (jb.kcols + 127) / 128;
      const int64_t k = (lt % tiles_k) * 128 + lane * 4;
      const int64_t r0 = (lt / tiles_k) * 32 + wy;
      if (k >= jb.kcols) continue;
      const bool full = k + 4 <= jb.kcols;
      float4 v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t r = r0 + 2 * i;
        if (r < jb.rows && full) v[i] = __ldcs(reinterpret_cast<const float4*>(jb.src + r * jb.lds + k));
      }
      int e[16];  // kModeF16x2 row exponents, loaded together ahead of the stores
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t r = r0 + 2 * i;
        e[i] = r < jb.rows ? splitdev::row_exp(p, r) : 0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t r = r0 + 2 * i;
        if (r >= jb.rows) break;
        if (full) {
          splitdev::split_store4(v[i], p, r, k, e[i]);
        } else {
          for (int64_t kk = k; kk < jb.kcols; ++kk)
            splitdev::split_store(__ldcs(jb.src + r * jb.lds + kk), p, r, kk, e[i]);
        }
      }
    } else {
      const int64_t tiles_k = (jb.kcols + 31) / 32;
      const int64_t k0 = (lt % tiles_k) * 32;
      const int64_t rb = (lt / tiles_k) * 128;
      const int64_t r = rb + lane * 4;
      split_bar();  // previous tile fully read
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int kl = wy + 2 * i;
        const int64_t k = k0 + kl;
        if (k >= jb.kcols) break;
        if (r + 4 <= jb.rows) {
          const float4 x = __ldcs(reinterpret_cast<const float4*>(jb.src + k * jb.lds + r));
          tile[kl][lane * 4 + 0] = x.x;
          tile[kl][lane * 4 + 1] = x.y;
          tile[kl][lane * 4 + 2] = x.z;
          tile[kl][lane * 4 + 3] = x.w;
        } else {
          for (int u = 0; u < 4; ++u)
            if (r + u < jb.rows) tile[kl][lane * 4 + u] = __ldcs(jb.src + k * jb.lds + r + u);
        }
      }
      split_bar();
      for (int rl = st >> 1; rl < 128; rl += 32) {
        const int64_t ro = rb + rl;
        if (ro >= jb.rows) break;
        const int e = splitdev::row_exp(p, ro);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kl = (st & 1) * 16 + 4 * q;
          const int64_t k = k0 + kl;
          if (k >= jb.kcols) break;
          if (k + 4 <= jb.kcols) {
            splitdev::split_store4(make_float4(tile[kl][rl], tile[kl + 1][rl], tile[kl + 2][rl], tile[kl + 3][rl]),
                                   p, ro, k, e);
          } else {
            for (int u = 0; k + u < jb.kcols; ++u) splitdev::split_store(tile[kl + u][rl], p, ro, k + u, e);
          }
        }
      }
    }
  }
}

// Numerics note.  The tensor core adds each MMA's products into the fp32
// accumulator with truncation (round toward zero), so the relative error of
// one TMEM accumulator grows linearly with the number of MMAs issued into it
// (measured ~2e-8 per MMA: 1.1e-4 at K=16384 without chunking).  The K loop is
// therefore cut into chunks of `kc_blocks` k-blocks: each chunk accumulates in
// a fresh TMEM buffer and the epilogue warps fold it into an fp32 register
// master with round-to-nearest adds, making the error K-independent.
// Stage layout (per CTA, 64 KB):
//   kModeTf32x3: [A_hi f32 16K | A_lo f32 16K | B_hi f32 16K | B_lo f32 16K]     (128B swizzle)
//   kModeMixed : [A_hi f32 16K | B_hi f32 16K | A_hi bf16 8K | A_lo bf16 8K |
//                 B_hi bf16 8K | B_lo bf16 8K]          (f32: 128B swizzle, bf16: 64B swizzle)
// The tensor-map array is in that order.
struct Maps {
  CUtensorMap m[6];
};

template <int CG, int MODE>
__global__ void __launch_bounds__(Cfg<CG>::kThreads, 1)
    tf32x3_gemm_kernel(const __grid_constant__ Maps maps, int K, int kc_blocks, EpiParams ep,
                       const __grid_constant__ SplitJobs sj) {
  using C = Cfg<CG>;
  using namespace ptx;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment is required by the 128B swizzle atoms.
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* full_bar = bars;                        // [kStages]
  uint64_t* empty_bar = bars + C::kStages;          // [kStages]
  uint64_t* cfull_bar = bars + 2 * C::kStages;      // [2] chunk accumulated
  uint64_t* cempty_bar = bars + 2 * C::kStages + 2; // [2] chunk drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 4);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t cta_rank = (CG == 2) ? cluster_ctarank() : 0u;
  const bool leader = cta_rank == 0;

  const int tiles_m = (ep.m + C::kUmmaM - 1) / C::kUmmaM;
  const int tiles_n = (ep.n + C::kUmmaN - 1) / C::kUmmaN;
  const int total_tiles = tiles_m * tiles_n;
  const int total_items = total_tiles * ep.ksplit;
  const int unit = blockIdx.x / CG;
  const int num_units = gridDim.x / CG;
  constexpr int kBK = stage_k<MODE>();
  const int num_kb = (K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&cfull_bar[a]), 1);
      mbar_init(smem_u32(&cempty_bar[a]), C::kEpiWarps * CG);
    }
    fence_barrier_init();
    for (int i = 0; i < (MODE == kModeMixed ? 6 : 4); ++i) prefetch_tmap(&maps.m[i]);
  }
  if (warp == 1) tmem_alloc<CG>(smem_u32(tmem_slot), C::kTmemCols);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pol = ep.l2_policy == 1   ? policy_evict_last()
                           : ep.l2_policy == 2 ? policy_evict_first()
                                               : policy_evict_normal();
      const int epochs = ep.lockstep > 0 ? (num_kb + ep.lockstep - 1) / ep.lockstep : 0;
      int wave = 0;
      for (int t = unit; t < total_items; t += num_units, ++wave) {
        // CTAs of this wave (the last wave may be partial)
        const int wave_ctas = CG * min(num_units, total_items - wave * num_units);
        int tile, split, kb_lo, kb_hi, mt, nt;
        item_range(t, total_tiles, num_kb, ep.ksplit, tile, split, kb_lo, kb_hi);
        tile_coords<CG>(tile, tiles_m, tiles_n, ep.group_m, mt, nt);
        const int arow = mt * C::kUmmaM + static_cast<int>(cta_rank) * C::kRowsPerCta;
        const int brow = nt * C::kUmmaN + static_cast<int>(cta_rank) * C::kRowsPerCta;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          if (epochs > 0 && kb % ep.lockstep == 0) {
            // Software lockstep: CTAs sharing A/B tiles read the same k-slices
            // at about the same time, so L2 serves the sharers instead of DRAM.
            // Arrive on this epoch, then let at most one epoch of slack build up.
            const int e = kb / ep.lockstep;
            unsigned* ctr = ep.sync + static_cast<int64_t>(wave) * epochs;
            atomicAdd(ctr + e, 1u);
            if (e > 0) {
              // bounded wait (~1e7 cycles): lockstep is a locality hint, never a
              // correctness dependency, so a CTA that is not co-resident cannot hang it
              const long long t0 = clock64();
              unsigned seen;
              do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ctr + e - 1) : "memory");
                if (seen >= static_cast<unsigned>(wave_ctas)) break;
                __nanosleep(64);
              } while (clock64() - t0 < 10000000ll);
            }
          }
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          uint8_t* st = smem + stage * C::kStageBytes;
          const uint32_t fb = smem_u32(&full_bar[stage]);
          const int kx = kb * kBK;
          uint32_t fb_tx = fb;  // barrier receiving the bytes (leader's for pairs)
          if constexpr (CG == 2)
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(fb_tx) : "r"(fb));
          if (leader) mbar_arrive_expect_tx(fb, CG * C::kStageBytes);
          auto load2 = [&](int i, uint32_t off, int x, int y) {
            if constexpr (CG == 1) tma_load_2d(&maps.m[i], smem_u32(st + off), fb_tx, x, y, pol);
            else tma_load_2d_cg2(&maps.m[i], smem_u32(st + off), fb_tx, x, y, pol);
          };
          // one operand tile (128 rows of M or N x 32 k): K-major = one box of
          // 128 rows; MN-major = 128-B slices along M/N (32 fp32 / 64 bf16
          // elements) of 32 k rows each, 4 KB apart
          auto load = [&](int i, uint32_t off, int row, bool mn, bool bf16) {
            if (!mn) {
              load2(i, off, kx, row);
            } else {
              const int w = bf16 ? 64 : 32;
#pragma unroll 1
              for (int c = 0; c < 128 / w; ++c) load2(i, off + c * 4096u, row + c * w, kx);
            }
          };
          const bool amn = ep.a_mn != 0, bmn = ep.b_mn != 0, amn16 = ep.a_mn16 != 0, bmn16 = ep.b_mn16 != 0;
          if constexpr (MODE == kModeF16x2) {
            // fp16 h0 / h1 tiles: 128 rows x 64 k (128 B), K-major
            load(0, 0, arow, false, false);
            load(1, C::kTileBytes, arow, false, false);
            load(2, 2 * C::kTileBytes, brow, false, false);
            load(3, 3 * C::kTileBytes, brow, false, false);
          } else if constexpr (MODE == kModeTf32x3) {
            load(0, 0, arow, amn, false);
            load(1, C::kTileBytes, arow, amn, false);
            load(2, 2 * C::kTileBytes, brow, bmn, false);
            load(3, 3 * C::kTileBytes, brow, bmn, false);
          } else {
            constexpr uint32_t h = C::kTileBytes / 2;  // bf16 tile: 128 rows x 64 B
            load(0, 0, arow, amn, false);
            load(1, C::kTileBytes, brow, bmn, false);
            load(2, 2 * C::kTileBytes, arow, amn16, true);
            load(3, 2 * C::kTileBytes + h, arow, amn16, true);
            load(4, 3 * C::kTileBytes, brow, bmn16, true);
            load(5, 3 * C::kTileBytes + h, brow, bmn16, true);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (leader && lane == 0) {
      const uint32_t idesc = idesc_tf32(C::kUmmaM, C::kUmmaN) | idesc_major(ep.a_mn, ep.b_mn);
      // descriptor of an operand tile and its advance (16-B units) per k8
      // (fp32) / k16 (bf16) step: K-major moves 32 B along the swizzled row,
      // MN-major moves 8 (16) k rows = 1024 (2048) B
      auto d32 = [](uint32_t a, int mn) { return mn ? sdesc_mn_sw128_32b(a) : sdesc_k_sw128(a); };
      auto d16 = [](uint32_t a, int mn) { return mn ? sdesc_mn_sw128(a) : sdesc_k_sw64(a); };
      const uint64_t ia32 = ep.a_mn ? 64 : 2, ib32 = ep.b_mn ? 64 : 2;
      const uint64_t ia16 = ep.a_mn16 ? 128 : 2, ib16 = ep.b_mn16 ? 128 : 2;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk_ctr = 0;
      for (int t = unit; t < total_items; t += num_units) {
        int tile, split, kb_lo, kb_hi;
        item_range(t, total_tiles, num_kb, ep.ksplit, tile, split, kb_lo, kb_hi);
        const int num_chunks = (kb_hi - kb_lo + kc_blocks - 1) / kc_blocks;
        for (int ch = 0; ch < num_chunks; ++ch, ++chunk_ctr) {
          const int buf = chunk_ctr & 1;
          mbar_wait(smem_u32(&cempty_bar[buf]), ((chunk_ctr >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * C::kAccCols);
          const int kb0 = kb_lo + ch * kc_blocks;
          const int kb1 = min(kb_hi, kb0 + kc_blocks);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(smem_u32(&full_bar[stage]), phase);
            tc_fence_after();
            const uint32_t s0 = smem_u32(smem + stage * C::kStageBytes);
            const uint32_t acc0 = (kb != kb0) ? 1u : 0u;
            if constexpr (MODE == kModeF16x2) {
              const uint32_t idesc16 = idesc_f16(C::kUmmaM, C::kUmmaN);
              const uint64_t a0 = sdesc_k_sw128(s0), a1 = sdesc_k_sw128(s0 + C::kTileBytes);
              const uint64_t b0 = sdesc_k_sw128(s0 + 2 * C::kTileBytes), b1 = sdesc_k_sw128(s0 + 3 * C::kTileBytes);
#pragma unroll
              for (int j = 0; j < kBK / 16; ++j) {
                // k16 step j (32 B along the swizzled row); small terms first, then h0*h0
                const uint64_t o = 2 * j;
                mma_bf16<CG>(d_tmem, a1 + o, b0 + o, idesc16, (acc0 | j) != 0);
                mma_bf16<CG>(d_tmem, a0 + o, b1 + o, idesc16, 1u);
                mma_bf16<CG>(d_tmem, a0 + o, b0 + o, idesc16, 1u);
              }
            } else if constexpr (MODE == kModeTf32x3) {
              const uint64_t ahi = d32(s0, ep.a_mn);
              const uint64_t alo = d32(s0 + C::kTileBytes, ep.a_mn);
              const uint64_t bhi = d32(s0 + 2 * C::kTileBytes, ep.b_mn);
              const uint64_t blo = d32(s0 + 3 * C::kTileBytes, ep.b_mn);
#pragma unroll
              for (int j = 0; j < C::kBK / 8; ++j) {
                // k8 step j; small terms first, then hi*hi
                const uint64_t oa = j * ia32, ob = j * ib32;
                mma_tf32<CG>(d_tmem, alo + oa, bhi + ob, idesc, (acc0 | j) != 0);
                mma_tf32<CG>(d_tmem, ahi + oa, blo + ob, idesc, 1u);
                mma_tf32<CG>(d_tmem, ahi + oa, bhi + ob, idesc, 1u);
              }
            } else {
              constexpr uint32_t h = C::kTileBytes / 2;
              const uint32_t idesc16 = idesc_bf16(C::kUmmaM, C::kUmmaN) | idesc_major(ep.a_mn16, ep.b_mn16);
              const uint64_t ahi = d32(s0, ep.a_mn);
              const uint64_t bhi = d32(s0 + C::kTileBytes, ep.b_mn);
              const uint64_t ah16 = d16(s0 + 2 * C::kTileBytes, ep.a_mn16);
              const uint64_t al16 = d16(s0 + 2 * C::kTileBytes + h, ep.a_mn16);
              const uint64_t bh16 = d16(s0 + 3 * C::kTileBytes, ep.b_mn16);
              const uint64_t bl16 = d16(s0 + 3 * C::kTileBytes + h, ep.b_mn16);
#pragma unroll
              for (int j = 0; j < C::kBK / 16; ++j) {
                // bf16 cross terms for k16 step j ...
                const uint64_t oa = j * ia16, ob = j * ib16;
                mma_bf16<CG>(d_tmem, ah16 + oa, bl16 + ob, idesc16, (acc0 | j) != 0);
                mma_bf16<CG>(d_tmem, al16 + oa, bh16 + ob, idesc16, 1u);
                // ... then hi*hi in tf32 for the same 16 k (two k8 MMAs)
                mma_tf32<CG>(d_tmem, ahi + 2 * j * ia32, bhi + 2 * j * ib32, idesc, 1u);
                mma_tf32<CG>(d_tmem, ahi + (2 * j + 1) * ia32, bhi + (2 * j + 1) * ib32, idesc, 1u);
              }
            }
            if constexpr (CG == 1) mma_commit(smem_u32(&empty_bar[stage]));
            else mma_commit_cg2(smem_u32(&empty_bar[stage]), 0x3);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
          if constexpr (CG == 1) mma_commit(smem_u32(&cfull_bar[buf]));
          else mma_commit_cg2(smem_u32(&cfull_bar[buf]), 0x3);
        }
      }
    }
  } else if (warp >= 2 + C::kEpiWarps) {
    // ------------------------------------------------------------ split warps
    if (sj.n > 0)
      run_split_jobs(sj, reinterpret_cast<float(*)[128 + 4]>(smem + C::kStages * C::kStageBytes + 256),
                     threadIdx.x - 32 * (2 + C::kEpiWarps), sj.phase_ctr != nullptr ? 2 : 0);
  } else {
    // ------------------------------------------------------------ epilogue
    const int e = warp - 2;
    const int q = warp % 4;           // TMEM lane quadrant this warp may access
    const int half = e / 4;           // which half of the accumulator columns
    const int col_off = half * C::kColsPerThread;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    uint32_t chunk_ctr = 0;
    for (int t = unit; t < total_items; t += num_units) {
      int tile, split, kb_lo, kb_hi, mt, nt;
      item_range(t, total_tiles, num_kb, ep.ksplit, tile, split, kb_lo, kb_hi);
      tile_coords<CG>(tile, tiles_m, tiles_n, ep.group_m, mt, nt);
      const int num_chunks = (kb_hi - kb_lo + kc_blocks - 1) / kc_blocks;
      // beta != 0: this thread's C row segment is read right after the last
      // chunk; pulling it into L2 a chunk earlier keeps those reads off the
      // DRAM latency path (the MMA has only two chunk buffers of slack)
      const int pf_chunk = (ep.c_prefetch > 0 && ep.read_c && ep.ksplit <= 1 && !ep.c_half)
                               ? max(0, num_chunks - ep.c_prefetch) : -1;
      float master[C::kColsPerThread];
#pragma unroll
      for (int j = 0; j < C::kColsPerThread; ++j) master[j] = 0.0f;
      for (int ch = 0; ch < num_chunks; ++ch, ++chunk_ctr) {
        const int buf = chunk_ctr & 1;
        if (ch == pf_chunk) {
          const int prow_i = mt * C::kUmmaM + static_cast<int>(cta_rank) * C::kRowsPerCta + q * 32 +
                             static_cast<int>(lane);
          const int pc0 = nt * C::kUmmaN + col_off;
          if (prow_i < ep.m) {
            const float* prow = ep.c + static_cast<int64_t>(prow_i) * ep.ldc + pc0;
#pragma unroll
            for (int l = 0; l < C::kColsPerThread / 32; ++l)
              if (pc0 + 32 * l < ep.n) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(prow + 32 * l));
          }
        }
        mbar_wait(smem_u32(&cfull_bar[buf]), (chunk_ctr >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + static_cast<uint32_t>(buf * C::kAccCols + col_off) + lane_addr;
#pragma unroll
        for (int g = 0; g < C::kColsPerThread / 16; ++g) {
          uint32_t v[16];
          tmem_ld_32x32b_x16(taddr + static_cast<uint32_t>(g * 16), v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) master[g * 16 + j] = __fadd_rn(master[g * 16 + j], __uint_as_float(v[j]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) mbar_arrive(smem_u32(&cempty_bar[buf]));
          else mbar_arrive_cluster(smem_u32(&cempty_bar[buf]), 0);
        }
      }
      const int row = mt * C::kUmmaM + static_cast<int>(cta_rank) * C::kRowsPerCta + q * 32 +
                      static_cast<int>(lane);
      if (row >= ep.m) continue;
      const int c0 = nt * C::kUmmaN + col_off;
      // kModeF16x2: undo the planes' power-of-two row scales as each value is
      // stored -- exact unless the result itself leaves the normal range
      const int ea = MODE == kModeF16x2 ? splitdev::f16x2_exp(__ldg(ep.a_max + row)) : 0;
      auto acc = [&](int j) -> float {
        if constexpr (MODE == kModeF16x2)
          return splitdev::unscale_pow2(master[j], -(ea + splitdev::f16x2_exp(__ldg(ep.b_max + c0 + j))));
        else
          return master[j];
      };
      // alpha / beta epilogue straight from the master registers; a split-K
      // item stores its raw partial (alpha = 1, no C) to its workspace slice
      const bool part = ep.ksplit > 1;
      float* const cbase = part ? ep.ws + static_cast<int64_t>(split) * ep.m * ep.n : ep.c;
      const int64_t ldc = part ? static_cast<int64_t>(ep.n) : ep.ldc;
      const float alpha = part ? 1.0f : ep.alpha;
      const int read_c = part ? 0 : ep.read_c;
      if (!part && ep.c_half) {
        // Half16 C: beta*C widened exactly, result rounded once (narrow_store)
        __half* hrow = reinterpret_cast<__half*>(cbase) + static_cast<int64_t>(row) * ldc + c0;
#pragma unroll
        for (int j = 0; j < C::kColsPerThread; ++j) {
          if (c0 + j < ep.n) {
            float v = __fmul_rn(alpha, acc(j));
            if (read_c) v = __fadd_rn(v, __fmul_rn(ep.beta, __half2float(hrow[j])));
            hrow[j] = __float2half_rn(v);
          }
        }
        continue;
      }
      float* crow = cbase + static_cast<int64_t>(row) * ldc + c0;
      const bool vec_ok = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(cbase) & 15) == 0);
      // C is read in groups of kEpiGroup float4 issued back to back (one
      // round trip per group, not per float4): with beta != 0 the epilogue
      // must not hold the chunk buffers longer than the MMA's two-chunk slack.
      constexpr int kEpiGroup = 4;
#pragma unroll
      for (int j0 = 0; j0 < C::kColsPerThread / 4; j0 += kEpiGroup) {
        const int cc0 = c0 + 4 * j0;
        if (cc0 >= ep.n) break;
        if (vec_ok && cc0 + 4 * kEpiGroup <= ep.n) {
          float4 cv[kEpiGroup];
          if (read_c) {
#pragma unroll
            for (int u = 0; u < kEpiGroup; ++u) cv[u] = __ldcs(reinterpret_cast<const float4*>(crow + 4 * (j0 + u)));
          }
#pragma unroll
          for (int u = 0; u < kEpiGroup; ++u) {
            const int j = j0 + u;
            float o[4];
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) o[q2] = __fmul_rn(alpha, acc(4 * j + q2));
            if (read_c) {
              o[0] = __fadd_rn(o[0], __fmul_rn(ep.beta, cv[u].x));
              o[1] = __fadd_rn(o[1], __fmul_rn(ep.beta, cv[u].y));
              o[2] = __fadd_rn(o[2], __fmul_rn(ep.beta, cv[u].z));
              o[3] = __fadd_rn(o[3], __fmul_rn(ep.beta, cv[u].w));
            }
            __stcs(reinterpret_cast<float4*>(crow + 4 * j), make_float4(o[0], o[1], o[2], o[3]));
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 4 * kEpiGroup; ++jj) {
            const int cc = cc0 + jj;
            if (cc < ep.n) {
              float v = __fmul_rn(alpha, acc(4 * j0 + jj));
              if (read_c) v = __fadd_rn(v, __fmul_rn(ep.beta, crow[4 * j0 + jj]));
              crow[4 * j0 + jj] = v;
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, C::kTmemCols);
  }
}

// All split jobs of a command in one launch (small, latency-bound commands:
// one kernel instead of one per piece, every piece's tiles in flight at once).
__global__ void __launch_bounds__(64) split_jobs_kernel(const __grid_constant__ SplitJobs sj, int phase) {
  __shared__ float tile[32][128 + 4];
  run_split_jobs(sj, tile, static_cast<int>(threadIdx.x), phase);
}

// C <- alpha*0 + beta*C for K == 0 (no tensor-core work).
__global__ void scale_c_kernel(float* c, int c_half, int64_t ldc, int m, int n, float alpha_zero,
                               float beta, int read_c) {
  const int64_t total = static_cast<int64_t>(m) * n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / n), cc = static_cast<int>(i % n);
    float o = __fmul_rn(alpha_zero, 0.0f);
    if (c_half) {
      __half* h = reinterpret_cast<__half*>(c);
      if (read_c) o = __fadd_rn(o, __fmul_rn(beta, __half2float(h[r * ldc + cc])));
      h[r * ldc + cc] = __float2half_rn(o);
    } else {
      if (read_c) o = __fadd_rn(o, __fmul_rn(beta, c[r * ldc + cc]));
      c[r * ldc + cc] = o;
    }
  }
}

// ------------------------------------------------------------------ host
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Operand plane of `rows` (M or N) x K elements.
//   K-major  (mn == false): [rows x K], row pitch `ld`; box 32 k x 128 rows --
//            fp32 with the 128-B swizzle, bf16 with the 64-B swizzle;
//   MN-major (mn == true) : [K x rows], row pitch `ld` (along M/N); box
//            128 B along M/N (32 fp32 / 64 bf16) x 32 k, 128-B swizzle (fp32:
//            of 32-B atoms, the only MN-major 32-bit layout tcgen05 reads).
// Out-of-range elements (edges of M, N, K) are zero-filled by the TMA.
int make_operand_map(CUtensorMap* map, const void* base, int64_t rows, int64_t k, int64_t ld,
                     bool bf16, bool mn, bool fp16 = false) {
  EncodeTiledFn enc = encode_fn();
  if (enc == nullptr) return -1;
  if (fp16) {
    // kModeF16x2 plane: K-major [rows x K] fp16, box 64 k (128 B) x 128 rows, 128-B swizzle
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    cuuint32_t box[2] = {64u, 128u};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
  }
  const int esz = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(mn ? rows : k), static_cast<cuuint64_t>(mn ? k : rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esz};
  cuuint32_t box[2] = {mn ? static_cast<cuuint32_t>(128 / esz) : 32u, mn ? 32u : 128u};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   !mn ? (bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B)
                       : (bf16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int device_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

int pick_cta_group(const Tf32x3Args& a) {
  if (a.cta_group != 0) return a.cta_group;
  // Pairs pay off once there are enough 256x256 tiles to fill the machine.
  const int64_t pair_tiles = ((a.m + 255) / 256) * ((a.n + 255) / 256);
  return pair_tiles >= 74 ? 2 : 1;
}

// Split-K factor: when the tiles cannot fill the machine (tall-skinny C, e.g.
// the FC layers' batch-wide strips), K is cut into S ranges of >= 512 so
// tiles x S work items cover the SMs; partials are summed in fixed order.
int pick_ksplit(const Tf32x3Args& a, int cg, int sms) {
  if (a.ksplit == 1 || a.k <= 0) return 1;
  const int64_t tiles = ((a.m + 128 * cg - 1) / (128 * cg)) * ((a.n + 128 * cg - 1) / (128 * cg));
  const int64_t units = sms / cg;
  const int64_t bk = a.mode == kModeF16x2 ? 64 : 32;
  const int64_t num_kb = (a.k + bk - 1) / bk;
  int64_t S = a.ksplit > 1 ? a.ksplit : (2 * tiles <= units ? std::min<int64_t>(units / tiles, num_kb / 16) : 1);
  S = std::max<int64_t>(1, std::min<int64_t>(S, 32));
  return static_cast<int>(S);
}

// out = alpha * sum_s ws[s] + beta * C, s ascending (deterministic).
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int S, int m, int n, float* c, int c_half,
                                     int64_t ldc, float alpha, float beta, int read_c) {
  const int64_t total = static_cast<int64_t>(m) * n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = __ldcs(ws + i);
    for (int sp = 1; sp < S; ++sp) acc = __fadd_rn(acc, __ldcs(ws + sp * total + i));
    const int64_t r = i / n, cc = i % n;
    float o = __fmul_rn(alpha, acc);
    if (c_half) {
      __half* h = reinterpret_cast<__half*>(c) + r * ldc + cc;
      if (read_c) o = __fadd_rn(o, __fmul_rn(beta, __half2float(*h)));
      *h = __float2half_rn(o);
    } else {
      float* f = c + r * ldc + cc;
      if (read_c) o = __fadd_rn(o, __fmul_rn(beta, *f));
      *f = o;
    }
  }
}

template <int CG, int MODE>
cudaError_t launch(const Tf32x3Args& a, cudaStream_t stream) {
  using C = Cfg<CG>;
  HostScope hs("tf32x3_gemm launch (host)");
  Maps maps;
  int bad = 0;
  const bool amn = a.a_mn != 0, bmn = a.b_mn != 0;
  const bool amn16 = (a.a_mn16 < 0 ? a.a_mn : a.a_mn16) != 0, bmn16 = (a.b_mn16 < 0 ? a.b_mn : a.b_mn16) != 0;
  if constexpr (MODE == kModeF16x2) {
    bad |= make_operand_map(&maps.m[0], a.a_hi16, a.m, a.k, a.lda16, false, false, true);
    bad |= make_operand_map(&maps.m[1], a.a_lo16, a.m, a.k, a.lda16, false, false, true);
    bad |= make_operand_map(&maps.m[2], a.b_hi16, a.n, a.k, a.ldb16, false, false, true);
    bad |= make_operand_map(&maps.m[3], a.b_lo16, a.n, a.k, a.ldb16, false, false, true);
  } else if constexpr (MODE == kModeTf32x3) {
    bad |= make_operand_map(&maps.m[0], a.a_hi, a.m, a.k, a.lda, false, amn);
    bad |= make_operand_map(&maps.m[1], a.a_lo, a.m, a.k, a.lda, false, amn);
    bad |= make_operand_map(&maps.m[2], a.b_hi, a.n, a.k, a.ldb, false, bmn);
    bad |= make_operand_map(&maps.m[3], a.b_lo, a.n, a.k, a.ldb, false, bmn);
  } else {
    bad |= make_operand_map(&maps.m[0], a.a_hi, a.m, a.k, a.lda, false, amn);
    bad |= make_operand_map(&maps.m[1], a.b_hi, a.n, a.k, a.ldb, false, bmn);
    bad |= make_operand_map(&maps.m[2], a.a_hi16, a.m, a.k, a.lda16, true, amn16);
    bad |= make_operand_map(&maps.m[3], a.a_lo16, a.m, a.k, a.lda16, true, amn16);
    bad |= make_operand_map(&maps.m[4], a.b_hi16, a.n, a.k, a.ldb16, true, bmn16);
    bad |= make_operand_map(&maps.m[5], a.b_lo16, a.n, a.k, a.ldb16, true, bmn16);
  }
  if (bad) return cudaErrorInvalidValue;
  // per-device opt-in to > 48 KB dynamic smem (idempotent; atomic so concurrent
  // host threads launching on different devices are well defined)
  static std::atomic<bool> attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(tf32x3_gemm_kernel<CG, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63].store(true, std::memory_order_release);
  }
  int sms = a.num_sms;
  if (sms <= 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = ((a.m + C::kUmmaM - 1) / C::kUmmaM) * ((a.n + C::kUmmaN - 1) / C::kUmmaN);
  int ksplit = pick_ksplit(a, CG, sms);
  if (ksplit > 1 && (a.ws == nullptr ||
                     a.ws_bytes < static_cast<size_t>(ksplit) * static_cast<size_t>(a.m * a.n) * sizeof(float)))
    ksplit = 1;  // no workspace: one item per tile
  int units = sms / CG;
  if (units > tiles * ksplit) units = tiles * ksplit;
  if (units < 1) units = 1;

  EpiParams ep{a.c, a.c_half, a.ldc, static_cast<int>(a.m), static_cast<int>(a.n), a.alpha, a.beta,
               a.read_c, a.group_m > 0 ? a.group_m : 8, a.l2_policy, a.lockstep, nullptr, ksplit, a.ws,
               a.a_mn, a.b_mn, amn16 ? 1 : 0, bmn16 ? 1 : 0, a.a_max, a.b_max,
               a.c_prefetch >= 0 ? a.c_prefetch : 0};
  // lockstep keeps the CTAs of a wave together; with a single wave there is
  // nothing to align (and no counters to clear)
  if (a.lockstep > 0 && a.sync != nullptr && ksplit == 1 && tiles > units) {
    const size_t need = tf32x3_sync_bytes(a);
    if (a.sync_bytes < need) return cudaErrorInvalidValue;
    ep.lockstep = a.lockstep;
    ep.sync = a.sync;
    cudaError_t e = cudaMemsetAsync(ep.sync, 0, need, stream);
    if (e != cudaSuccess) return e;
  } else {
    ep.lockstep = 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * CG);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int64_t flush = a.flush_k > 0 ? a.flush_k : tf32x3_default_flush_k(a.mode, a.k_total > 0 ? a.k_total : a.k);
  constexpr int kBK = stage_k<MODE>();
  const int kc_blocks = static_cast<int>(std::max<int64_t>(1, (flush + kBK - 1) / kBK));
  SplitJobs sj;
  if (a.split != nullptr) sj = *a.split;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tf32x3_gemm_kernel<CG, MODE>, maps, static_cast<int>(a.k),
                                     kc_blocks, ep, sj);
  if (e != cudaSuccess || ksplit == 1) return e;
  const int64_t total = a.m * a.n;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * sms));
  splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(a.ws, ksplit, static_cast<int>(a.m), static_cast<int>(a.n),
                                                   a.c, a.c_half, a.ldc, a.alpha, a.beta, a.read_c);
  return cudaGetLastError();
}

}  // namespace

cudaError_t stream_write_flag(cudaStream_t stream, unsigned* addr, unsigned value) {
  using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WriteValueFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<WriteValueFn>(nullptr);
    return reinterpret_cast<WriteValueFn>(p);
  }();
  if (fn == nullptr) return cudaErrorNotSupported;
  return fn(stream, reinterpret_cast<CUdeviceptr>(addr), value, 0) == CUDA_SUCCESS ? cudaSuccess
                                                                                    : cudaErrorUnknown;
}

cudaError_t split_jobs(const SplitJobs& jobs, cudaStream_t stream) {
  if (jobs.n <= 0 || jobs.t_end <= jobs.t_begin) return cudaSuccess;
  for (int i = 0; i < jobs.n; ++i)
    if (jobs.job[i].flag != nullptr || !split_job_fusable(jobs.job[i])) return cudaErrorInvalidValue;
  const int64_t tiles = jobs.t_end - jobs.t_begin;
  const int blocks = static_cast<int>(std::min<int64_t>(tiles, 148 * 16));
  if (jobs.job[0].rmax != nullptr) {  // kModeF16x2: row maxima first (separate launch = grid-wide order)
    split_jobs_kernel<<<blocks, 64, 0, stream>>>(jobs, 1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  split_jobs_kernel<<<blocks, 64, 0, stream>>>(jobs, 0);
  return cudaGetLastError();
}

int64_t tf32x3_default_flush_k(int mode, int64_t k_total) {
  if (k_total <= 512) return 32;
  if (k_total <= 2048) return 64;
  if (mode == kModeTf32x3) return 128;  // 3xTF32: 128 runs as fast as 256
  if (mode == kModeF16x2) return k_total <= 8192 ? 128 : 256;  // 24 / 48 MMAs per chunk
  return k_total <= 8192 ? 128 : 256;
}

int64_t split_job_tiles(const SplitJob& j) {
  if (j.rows <= 0 || j.kcols <= 0) return 0;
  return j.trans ? ((j.kcols + 31) / 32) * ((j.rows + 127) / 128) : ((j.rows + 31) / 32) * ((j.kcols + 127) / 128);
}

bool split_job_fusable(const SplitJob& j) {
  auto al = [](const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
  if (j.rmax != nullptr)  // kModeF16x2: fp16 h0 / h1 in hi16 / lo16
    return j.src != nullptr && al(j.src, 16) && (j.lds & 3) == 0 && j.hi16 != nullptr && al(j.hi16, 8) &&
           al(j.lo16, 8) && (j.ldo16 & 3) == 0;
  return j.src != nullptr && al(j.src, 16) && (j.lds & 3) == 0 && j.hi != nullptr && al(j.hi, 16) &&
         (j.ldo & 3) == 0 && (j.lo == nullptr || al(j.lo, 16)) &&
         (j.hi16 == nullptr || (al(j.hi16, 8) && al(j.lo16, 8) && (j.ldo16 & 3) == 0));
}

size_t tf32x3_splitk_bytes(const Tf32x3Args& a) {
  if (a.m <= 0 || a.n <= 0 || a.k <= 0) return 0;
  const int cg = pick_cta_group(a);
  const int sms = a.num_sms > 0 ? a.num_sms : device_sms();
  const int S = pick_ksplit(a, cg, sms);
  return S > 1 ? static_cast<size_t>(S) * static_cast<size_t>(a.m * a.n) * sizeof(float) : 0;
}

size_t tf32x3_sync_bytes(const Tf32x3Args& a) {
  if (a.lockstep <= 0 || a.m <= 0 || a.n <= 0 || a.k <= 0) return 0;
  const int64_t tiles = ((a.m + 127) / 128) * ((a.n + 127) / 128);  // upper bound (1-CTA tiles)
  const int64_t num_kb = (a.k + 31) / 32;
  const int64_t epochs = (num_kb + a.lockstep - 1) / a.lockstep;
  return static_cast<size_t>(tiles * epochs) * sizeof(unsigned);  // waves <= tiles
}

cudaError_t tf32x3_gemm(const Tf32x3Args& a, cudaStream_t stream) {
  if (a.split != nullptr && a.split->n > 0 && (a.m <= 0 || a.n <= 0 || a.k <= 0))
    return cudaErrorInvalidValue;  // fused split work needs a real GEMM launch to ride on
  if (a.m <= 0 || a.n <= 0) return cudaSuccess;
  if (a.k <= 0) {
    const int64_t total = a.m * a.n;
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    scale_c_kernel<<<blocks, 256, 0, stream>>>(a.c, a.c_half, a.ldc, static_cast<int>(a.m),
                                               static_cast<int>(a.n), a.alpha, a.beta, a.read_c);
    return cudaGetLastError();
  }
  // TMA needs 16-B aligned bases and pitches.
  auto mis = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
  if ((a.lda & 3) || (a.ldb & 3) || mis(a.a_hi) || mis(a.b_hi)) return cudaErrorMisalignedAddress;
  if (a.mode == kModeTf32x3 && (mis(a.a_lo) || mis(a.b_lo))) return cudaErrorMisalignedAddress;
  if (a.mode == kModeMixed && ((a.lda16 & 7) || (a.ldb16 & 7) || mis(a.a_hi16) || mis(a.a_lo16) ||
                               mis(a.b_hi16) || mis(a.b_lo16)))
    return cudaErrorMisalignedAddress;
  const int cg = pick_cta_group(a);
  if (a.mode == kModeF16x2) {
    if (a.a_mn || a.b_mn || a.a_max == nullptr || a.b_max == nullptr) return cudaErrorInvalidValue;
    if ((a.lda16 & 7) || (a.ldb16 & 7) || mis(a.a_hi16) || mis(a.a_lo16) || mis(a.b_hi16) || mis(a.b_lo16))
      return cudaErrorMisalignedAddress;
    return cg == 2 ? launch<2, kModeF16x2>(a, stream) : launch<1, kModeF16x2>(a, stream);
  }
  if (a.mode == kModeMixed) return cg == 2 ? launch<2, kModeMixed>(a, stream) : launch<1, kModeMixed>(a, stream);
  return cg == 2 ? launch<2, kModeTf32x3>(a, stream) : launch<1, kModeTf32x3>(a, stream);
}

}  // namespace dm
