// KV codec spec shared by the codec kernels.
// Host-side plan/layout arithmetic and device bit helpers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kvt_b200.h"

namespace kvt {

constexpr int kD = 128;      // head dim (one 256-byte bf16 row)
constexpr int kChunks = 16;  // canonical reduction: 16 chunks of 8 channels

inline double eff_bytes(int bits) { return bits >= 16 ? 1.0 : double(bits) / 16.0 + 1.0 / 64.0; }

inline int64_t al256(int64_t x) { return (x + 255) & ~int64_t(255); }

inline void blob_map(const kvt_kv_shape& s, const kvt_codec_cfg& c, kvt_blob_map* o) {
  const int64_t S = int64_t(s.L) * s.H, k = c.keep, D = s.D;
  std::memset(o, 0, sizeof(*o));
  int64_t off = 0;
  o->idx_off = off;
  o->idx_bytes = 4 * S * k;
  off = al256(off + o->idx_bytes);
  if (c.bits == 16) {
    o->kcode_off = off;
    o->kcode_bytes = 2 * S * k * D;
    off = al256(off + o->kcode_bytes);
    o->vcode_off = off;
    o->vcode_bytes = o->kcode_bytes;
    off = al256(off + o->vcode_bytes);
  } else {
    const int64_t wpr = D * c.bits / 32, ng = (k + KVT_QGROUP - 1) / KVT_QGROUP;
    o->kcode_off = off;
    o->kcode_bytes = 4 * S * k * wpr;
    off = al256(off + o->kcode_bytes);
    o->kparam_bytes = 2 * S * ng * D;
    o->kscale_off = off;
    off = al256(off + o->kparam_bytes);
    o->kzero_off = off;
    off = al256(off + o->kparam_bytes);
    o->vcode_off = off;
    o->vcode_bytes = o->kcode_bytes;
    off = al256(off + o->vcode_bytes);
    o->vparam_bytes = 2 * S * k;
    o->vscale_off = off;
    off = al256(off + o->vparam_bytes);
    o->vzero_off = off;
    off = al256(off + o->vparam_bytes);
  }
  o->total_bytes = off;
}

#ifdef __CUDACC__
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Synthetic bf16 element (integer-only; identical on the CPU oracle).
__device__ __forceinline__ uint16_t synth_bf16(uint64_t seed, uint64_t ctx, uint64_t idx, bool outlier) {
  const uint64_t z = mix64(seed * 0x9e3779b97f4a7c15ull + ctx * 0xc2b2ae3d27d4eb4full + idx * 0x9e3779b97f4a7c15ull);
  const uint32_t sign = uint32_t(z & 1u), mant = uint32_t((z >> 1) & 0x7fu);
  const uint32_t e = 124u + uint32_t((z >> 8) & 3u) + (outlier ? 3u : 0u);
  return uint16_t((sign << 15) | (e << 7) | mant);
}

__device__ __forceinline__ float bf2f(uint32_t bits16) { return __uint_as_float(bits16 << 16); }

// Orderable key: larger float -> larger key; -0 == +0.
__device__ __forceinline__ uint32_t score_key(float f) {
  if (f == 0.0f) f = 0.0f;
  const uint32_t x = __float_as_uint(f);
  return (x & 0x80000000u) ? ~x : (x | 0x80000000u);
}

struct QParam {
  float sf, zf, inv;
  uint16_t s16, z16;
};

// asymmetric min/max group parameters stored as fp16 scale + zero
__device__ __forceinline__ QParam make_param(float mn, float mx, int bits) {
  QParam p;
  mn = __fadd_rn(mn, 0.0f);  // -0 -> +0: the result does not depend on which zero min/max kept
  mx = __fadd_rn(mx, 0.0f);
  const float levels = float((1 << bits) - 1);
  const float scale = __fdiv_rn(__fsub_rn(mx, mn), levels);
  const __half hs = __float2half_rn(scale), hz = __float2half_rn(mn);
  p.s16 = __half_as_ushort(hs);
  p.z16 = __half_as_ushort(hz);
  p.sf = __half2float(hs);
  p.zf = __half2float(hz);
  p.inv = p.sf > 0.0f ? __frcp_rn(p.sf) : 0.0f;
  return p;
}

__device__ __forceinline__ uint32_t quant(float x, const QParam& p, int bits) {
  float r = rintf(__fmul_rn(__fsub_rn(x, p.zf), p.inv));
  const float hi = float((1 << bits) - 1);
  if (!(r >= 0.0f)) r = 0.0f;
  if (r > hi) r = hi;
  return uint32_t(r);
}

// Two codes at once with packed fp32x2 arithmetic (FADD2/FMUL2; each lane
// rounds exactly like the scalar ops): clamp(rint((x - z) * inv), 0, hi).
// Clamping before rounding is equivalent because 0 and hi are integers;
// fmaxf maps NaN to 0 like quant(). rint = add 1.5*2^23 (round-half-even).
__device__ __forceinline__ void quant2(float x0, float x1, float z0, float z1, float i0, float i1, float hi,
                                       uint32_t& c0, uint32_t& c1) {
  float2 y = __fmul2_rn(__fadd2_rn(make_float2(x0, x1), make_float2(-z0, -z1)), make_float2(i0, i1));
  y.x = fminf(fmaxf(y.x, 0.0f), hi);
  y.y = fminf(fmaxf(y.y, 0.0f), hi);
  const float2 r = __fadd2_rn(y, make_float2(12582912.0f, 12582912.0f));
  c0 = __float_as_uint(r.x) - 0x4B400000u;
  c1 = __float_as_uint(r.y) - 0x4B400000u;
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// packed bf16x2 min (exact); max is taken as min of negated values
__device__ __forceinline__ uint32_t bmin2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmin2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ uint16_t dequant_bf16(uint32_t code, float sf, float zf) {
  const float y = __fadd_rn(__fmul_rn(float(code), sf), zf);
  return __bfloat16_as_ushort(__float2bfloat16_rn(y));
}
#endif

}  // namespace kvt
