// ted_vec.cuh -- bf16 vector helpers shared by the HBM-bound kernels.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "ted_internal.h"

namespace ted {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float2 bf2_to_f2(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}
__device__ __forceinline__ uint32_t f2_to_bf2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  float2 t;
  t = bf2_to_f2(u.x); f[0] = t.x; f[1] = t.y;
  t = bf2_to_f2(u.y); f[2] = t.x; f[3] = t.y;
  t = bf2_to_f2(u.z); f[4] = t.x; f[5] = t.y;
  t = bf2_to_f2(u.w); f[6] = t.x; f[7] = t.y;
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  u.x = f2_to_bf2(f[0], f[1]);
  u.y = f2_to_bf2(f[2], f[3]);
  u.z = f2_to_bf2(f[4], f[5]);
  u.w = f2_to_bf2(f[6], f[7]);
  return u;
}
// streaming 16-byte load that does not allocate in L1
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// AdamW on one element (optimizer.cpp:94-100): m = b1 m + (1-b1) g, v = b2 v + (1-b2) g^2,
// p -= lr (m c1 / (sqrt(v c2) + eps) + wd p) with c1, c2 the bias corrections.  Every AdamW
// kernel (the fused wgrad epilogue and the standalone ones) uses this one expression, so
// fused and unfused steps agree bit for bit.  IEEE sqrt and division: the SFU-approximate
// pair (sqrt.approx + rcp.approx, a third of the instructions) measured 3-4 % SLOWER in the
// fused wgrad epilogue inside the power-capped step (tools/ab_lib.sh, same box), and again
// 3 % slower for the CTA-pair kernel alone (tools/wgrad_power.sh: 7.23 vs 7.03 ms per
// launch, although its SM clock settled higher, 1150 vs 1027 MHz).
__device__ __forceinline__ void adamw_elem(float& p, float& m, float& v, float g, const AdamK& k,
                                           float c1, float c2) {
  m = k.b1 * m + k.omb1 * g;
  v = k.b2 * v + (k.omb2 * g) * g;
  p -= k.lr * ((m * c1) / (sqrtf(v * c2) + k.eps) + k.wd * p);
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

}  // namespace
// Reduce-scatter of 32 per-lane partial values: afterwards lane l holds the warp total of
// value index l (31 shuffles instead of 32 x 5).
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const float send = upper ? v[i] : v[i + off];
      const float keep = upper ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

}  // namespace ted
