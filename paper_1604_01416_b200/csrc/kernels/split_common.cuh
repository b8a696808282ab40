// Device helpers shared by the split kernels and the GEMM's fused split warps:
// fp32 -> tf32 (RNE) hi / lo and bf16 hi / lo planes, K-major.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dm {
namespace splitdev {

__device__ __forceinline__ float tf32_rne(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) != 0x7f800000u) u += 0xFFFu + ((u >> 13) & 1u);
  return __uint_as_float(u & 0xFFFFE000u);
}

struct Planes {
  float* hi;
  float* lo;            // tf32 lo (kModeTf32x3) or null
  __nv_bfloat16* hi16;  // bf16(hi) (kModeMixed) or null
  __nv_bfloat16* lo16;
  int64_t ldo, ldo16;
};

__device__ __forceinline__ void split_store(float x, const Planes& p, int64_t r, int64_t k) {
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
__device__ __forceinline__ void split_store4(float4 x, const Planes& p, int64_t r, int64_t k) {
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
