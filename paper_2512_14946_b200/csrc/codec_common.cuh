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
  if (c.keep == s.T && c.bits == 16) {  // identity: the source KV is the compressed chunk
    o->identity = 1;
    return;
  }
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
  bool fast;  // |(x - zf) * inv| <= 16000 for every x of the group: int16-lane fast path is exact
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
  // x in [mn, mx] -> |fl(x - zf)| <= b and |y| <= fl(b * inv) (monotone rounding); NaN/inf -> slow path
  const float b = fmaxf(fabsf(__fsub_rn(mn, p.zf)), fabsf(__fsub_rn(mx, p.zf)));
  p.fast = __fmul_rn(b, p.inv) <= 16000.0f;
  return p;
}

// code = clamp(rint(exact((x - zf) * inv)), 0, 2^b - 1) (oracle quant): the
// difference is one fp32 op, the product is exact in FP64 and rounded once.
// Valid for any input (the slow path of the fast lanes below).
__device__ __forceinline__ uint32_t quant_exact(float x, float zf, float inv, int bits) {
  const double r = rint(double(__fsub_rn(x, zf)) * double(inv));
  const double hi = double((1 << bits) - 1);
  return r >= 0.0 ? uint32_t(r > hi ? hi : r) : 0u;
}

// Fast path of quant_exact for 8 channels (one 16-byte bf16 chunk, words
// q = channel pairs (2q, 2q+1)): one packed fp32x2 subtract and one fused
// multiply-add with 1.5 * 2^23 (= rint of the exact product, |y| < 2^22),
// then both codes clamped as int16 lanes (min + relu, one op). Lane word q: code 2q in bits
// 0..15, code 2q+1 in bits 16..31. Exact when QParam::fast holds.
template <int BITS>
__device__ __forceinline__ void quant8_fast(const uint4& v, const float2 (&nz)[4], const float2 (&iv)[4],
                                            uint32_t (&p)[4]) {
  constexpr uint32_t hi2 = ((1u << BITS) - 1u) * 0x00010001u;
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 d = __fadd2_rn(make_float2(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u)), nz[q]);
    const float2 r = __ffma2_rn(d, iv[q], make_float2(12582912.0f, 12582912.0f));
    const uint32_t c = __byte_perm(__float_as_uint(r.x), __float_as_uint(r.y), 0x5410);
    p[q] = __vimin_s16x2_relu(c, hi2);  // max(min(c, 2^b - 1), 0) per int16 lane, one instruction
  }
}
// same lane layout through quant_exact (any parameters)
template <int BITS>
__device__ __forceinline__ void quant8_exact(const uint4& v, const float (&z)[8], const float (&iv)[8],
                                             uint32_t (&p)[4]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    p[q] = quant_exact(__uint_as_float(w[q] << 16), z[2 * q], iv[2 * q], BITS) |
           (quant_exact(__uint_as_float(w[q] & 0xffff0000u), z[2 * q + 1], iv[2 * q + 1], BITS) << 16);
}

// 8 codes (lane words) -> the blob's bit packing of those 8 channels:
// BITS 8: two words (byte e = channel e); 4: one word (nibble e); 2: the
// low 16 bits (2-bit field e).
template <int BITS>
__device__ __forceinline__ uint2 pack8(const uint32_t (&p)[4]) {
  if (BITS == 8) return make_uint2(__byte_perm(p[0], p[1], 0x6420), __byte_perm(p[2], p[3], 0x6420));
  // codes sit in 16-bit lanes (code 2q in bits 0.., code 2q+1 in bits 16..):
  // shifted adds interleave them without overlapping bits (LEA), then one
  // x + (x >> k) (LEA.HI) folds the high lanes down next to the low ones
  if (BITS == 4) {
    const uint32_t x = p[0] + (p[1] << 8), y = p[2] + (p[3] << 8);  // codes 0,2 | 1,3 (and 4,6 | 5,7)
    const uint32_t xs = x + (x >> 12), ys = y + (y >> 12);          // low 16 bits: nibbles 0..3 (4..7)
    return make_uint2(__byte_perm(xs, ys, 0x5410), 0u);
  }
  const uint32_t x = p[0] + (p[1] << 4), y = p[2] + (p[3] << 4);
  const uint32_t z = x + (y << 8);  // codes 0,2,4,6 at bits 0,4,8,12; 1,3,5,7 at 16,20,24,28
  return make_uint2((z + (z >> 14)) & 0xffffu, 0u);
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
