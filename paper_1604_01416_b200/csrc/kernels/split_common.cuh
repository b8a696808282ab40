// Device helpers shared by the split kernels and the GEMM's fused split warps:
// fp32 -> tf32 (RNE) hi / lo and bf16 hi / lo planes, K-major; or, in the
// scaled 2xFP16 scheme (kModeF16x2), fp16 h0 / h1 planes of x * 2^e with e
// per plane row from the row's |x| maximum.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dm {
namespace splitdev {

__device__ __forceinline__ float tf32_rne(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) != 0x7f800000u) u += 0xFFFu + ((u >> 13) & 1u);
  return __uint_as_float(u & 0xFFFFE000u);
}

// ---- scaled 2xFP16 split (kModeF16x2)
// Row r of a plane is scaled by 2^e(r), e = 14 - floor(log2(max_k |x[r][k]|)),
// so the row maximum lands in [2^14, 2^15) (fp16 max 65504), then
//   h0 = fp16_rn(x 2^e),  h1 = fp16_rn(x 2^e - h0)      (the difference is exact)
// -- an 11-bit + 11-bit pair like 3xTF32's tf32 hi / lo, with the same three
// products (h0 h0 + h0 h1 + h1 h0, h1 h1 ~2^-22 dropped), but on the fp16
// tensor-core rate (2x tf32).  The epilogue multiplies by 2^-(e_A(i) + e_B(j)).
// The maximum is kept as the bits of a non-negative float (atomicMax on the
// unsigned bits orders non-negative floats); a zero / non-finite row is not
// scaled (e = 0).
__device__ __forceinline__ int f16x2_exp(unsigned maxbits) {
  if (maxbits == 0u || maxbits >= 0x7f800000u) return 0;
  const int ef = static_cast<int>(maxbits >> 23);
  const int lg = ef != 0 ? ef - 127 : (31 - __clz(static_cast<int>(maxbits))) - 149;  // floor(log2(max))
  return 14 - lg;  // in [-113, 163]
}
// 2^i as a float, i in [-126, 127]
__device__ __forceinline__ float pow2i(int i) { return __int_as_float((i + 127) << 23); }
// x * 2^e for e in [-252, 254], exact whenever the result is a normal float
// (two power-of-two factors, both within the normal range)
__device__ __forceinline__ float scale_pow2(float x, int e) {
  const int e1 = e >> 1;
  return __fmul_rn(__fmul_rn(x, pow2i(e1)), pow2i(e - e1));
}
// acc * 2^s for s in [-326, 226] (the epilogue's -(e_A + e_B)): one multiply in
// the common range, else three factors of one sign (no spurious overflow)
__device__ __forceinline__ float unscale_pow2(float acc, int s) {
  if (s >= -126 && s <= 127) return __fmul_rn(acc, pow2i(s));
  const int s1 = max(-100, min(100, s));
  const int s2 = max(-100, min(100, s - s1));
  return __fmul_rn(__fmul_rn(__fmul_rn(acc, pow2i(s1)), pow2i(s2)), pow2i(s - s1 - s2));
}

struct Planes {
  float* hi;
  float* lo;            // tf32 lo (kModeTf32x3) or null
  __nv_bfloat16* hi16;  // bf16(hi) (kModeMixed) or null
  __nv_bfloat16* lo16;
  int64_t ldo, ldo16;
  // kModeF16x2: fp16 h0 / h1 planes (pitch ldo16) and the per-row |x| maxima
  // (hi / lo / hi16 / lo16 null)
  __half* h0 = nullptr;
  __half* h1 = nullptr;
  const unsigned* rmax = nullptr;
};

__device__ __forceinline__ void split_store_f16x2(float x, int e, const Planes& p, int64_t r, int64_t k) {
  const float xs = scale_pow2(x, e);
  const __half a = __float2half_rn(xs);
  p.h0[r * p.ldo16 + k] = a;
  p.h1[r * p.ldo16 + k] = __float2half_rn(xs - __half2float(a));
}

__device__ __forceinline__ void split_store4_f16x2(float4 x, int e, const Planes& p, int64_t r, int64_t k) {
  const float v[4] = {scale_pow2(x.x, e), scale_pow2(x.y, e), scale_pow2(x.z, e), scale_pow2(x.w, e)};
  __half2 a[2], b[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    a[u] = __floats2half2_rn(v[2 * u], v[2 * u + 1]);
    const float2 af = __half22float2(a[u]);
    b[u] = __floats2half2_rn(v[2 * u] - af.x, v[2 * u + 1] - af.y);
  }
  uint2 hv, lv;
  hv.x = *reinterpret_cast<uint32_t*>(&a[0]);
  hv.y = *reinterpret_cast<uint32_t*>(&a[1]);
  lv.x = *reinterpret_cast<uint32_t*>(&b[0]);
  lv.y = *reinterpret_cast<uint32_t*>(&b[1]);
  __stcs(reinterpret_cast<uint2*>(p.h0 + r * p.ldo16 + k), hv);
  __stcs(reinterpret_cast<uint2*>(p.h1 + r * p.ldo16 + k), lv);
}

// Scale exponent of plane row r (kModeF16x2; 0 otherwise).  Callers load it
// once per row, ahead of the row's stores: an L2 round trip per store would
// serialise the split behind the loads.
__device__ __forceinline__ int row_exp(const Planes& p, int64_t r) {
  return p.rmax != nullptr ? f16x2_exp(__ldcg(p.rmax + r)) : 0;
}

// e: row_exp(p, r)
__device__ __forceinline__ void split_store(float x, const Planes& p, int64_t r, int64_t k, int e) {
  if (p.rmax != nullptr) return split_store_f16x2(x, e, p, r, k);
  const float h = tf32_rne(x);
  const float l = x - h;  // exact
  __stcs(p.hi + r * p.ldo + k, h);
  if (p.lo) __stcs(p.lo + r * p.ldo + k, tf32_rne(l));
  if (p.hi16) {
    p.hi16[r * p.ldo16 + k] = __float2bfloat16_rn(h);
    p.lo16[r * p.ldo16 + k] = __float2bfloat16_rn(l);
  }
}

// four consecutive k of one row (16-B / 8-B aligned plane rows)
__device__ __forceinline__ void split_store4(float4 x, const Planes& p, int64_t r, int64_t k, int e) {
  if (p.rmax != nullptr) return split_store4_f16x2(x, e, p, r, k);
  const float v[4] = {x.x, x.y, x.z, x.w};
  float h[4], l[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    h[u] = tf32_rne(v[u]);
    l[u] = v[u] - h[u];
  }
  // planes are consumed by the next GEMM's TMA, GBs later: stream them past L2
  __stcs(reinterpret_cast<float4*>(p.hi + r * p.ldo + k), make_float4(h[0], h[1], h[2], h[3]));
  if (p.lo)
    __stcs(reinterpret_cast<float4*>(p.lo + r * p.ldo + k),
           make_float4(tf32_rne(l[0]), tf32_rne(l[1]), tf32_rne(l[2]), tf32_rne(l[3])));
  if (p.hi16) {
    __nv_bfloat162 a0 = __floats2bfloat162_rn(h[0], h[1]), a1 = __floats2bfloat162_rn(h[2], h[3]);
    __nv_bfloat162 b0 = __floats2bfloat162_rn(l[0], l[1]), b1 = __floats2bfloat162_rn(l[2], l[3]);
    uint2 hv, lv;
    hv.x = *reinterpret_cast<uint32_t*>(&a0);
    hv.y = *reinterpret_cast<uint32_t*>(&a1);
    lv.x = *reinterpret_cast<uint32_t*>(&b0);
    lv.y = *reinterpret_cast<uint32_t*>(&b1);
    __stcs(reinterpret_cast<uint2*>(p.hi16 + r * p.ldo16 + k), hv);
    __stcs(reinterpret_cast<uint2*>(p.lo16 + r * p.ldo16 + k), lv);
  }
}

}  // namespace splitdev
}  // namespace dm
