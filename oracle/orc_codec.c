/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle of the KV codec.
 *
 * PARITY UNPINNED: the reference has no codec (SPEC.md:15 puts the
 * keydiff/knorm/snapkv kernels out of scope; proj/include/kvtier/core.hpp:
 * 26-27 models a method as a label + size ratio). This file restates the
 * builder-defined codec spec of DESIGN.md §"Codec spec" (derived from
 * PAPER.md:636-638 for the scorers and PAPER.md:798,829-831 for KIVI-style
 * quantisation) and is pinned by the known-answer tests in
 * tests/test_codec_oracle.py, not by reference vectors.
 *
 * Every rounding step is spelled out so the CUDA path can match it
 * bit-for-bit (spec v2; snapkv v4): fp32 dot products with explicit
 * fmaf chains in the canonical chunk-then-butterfly order, 2^-21
 * fixed-point int64 accumulation for keydiff's mean direction, snapkv as
 * exact int8 x int8 logits with an integer-shift softmax, fp32 IEEE ops
 * (no contraction: built with -ffp-contract=off) for quantisation,
 * round-half-even everywhere.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "orc_common.h"

/* ------------------------------------------------------------- bit utils */

static float bf2f(uint16_t b) {
  uint32_t x = (uint32_t)b << 16;
  float f;
  memcpy(&f, &x, 4);
  return f;
}

static uint16_t f2bf(float f) { /* round to nearest even */
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((x >> 16) | 0x40);
  x += 0x7fffu + ((x >> 16) & 1u);
  return (uint16_t)(x >> 16);
}

static uint32_t rne_shift(uint32_t v, int s) { /* round v / 2^s to nearest even */
  if (s <= 0) return v;
  if (s >= 32) return 0;
  uint32_t q = v >> s, r = v & ((1u << s) - 1u), half = 1u << (s - 1);
  if (r > half || (r == half && (q & 1u))) ++q;
  return q;
}

static uint16_t f2h(float f) { /* IEEE binary16, round to nearest even */
  uint32_t x;
  memcpy(&x, &f, 4);
  uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  uint32_t a = x & 0x7fffffffu;
  if (a > 0x7f800000u) return sign | 0x7e00u;
  if (a >= 0x477ff000u) return sign | 0x7c00u; /* >= 65520 -> inf */
  if (a >= 0x38800000u) {                      /* normal half */
    uint32_t h = (a >> 13) - (112u << 10);
    uint32_t r = a & 0x1fffu;
    if (r > 0x1000u || (r == 0x1000u && (h & 1u))) ++h;
    return (uint16_t)(sign | h);
  }
  int e = (int)(a >> 23);
  if (e == 0) return sign; /* float subnormal: far below half's range */
  uint32_t mant = (a & 0x7fffffu) | 0x800000u; /* value = mant * 2^(e-150) */
  return (uint16_t)(sign | rne_shift(mant, 126 - e));
}

static float h2f(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu, x;
  if (e == 0) {
    if (m == 0) {
      x = sign;
    } else { /* subnormal: m * 2^-24 */
      float f = (float)m * 5.9604644775390625e-08f;
      memcpy(&x, &f, 4);
      x |= sign;
    }
  } else if (e == 31) {
    x = sign | 0x7f800000u | (m << 13);
  } else {
    x = sign | ((e + 112u) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &x, 4);
  return f;
}

/* ---------------------------------------------------------- plan/layout */

#define D_HEAD 128
#define NCHUNK 16 /* canonical reduction: 16 chunks of 8 channels */

static double eff_bytes(int bits) { /* retained bytes per bf16 byte */
  return bits >= 16 ? 1.0 : (double)bits / 16.0 + 1.0 / 64.0;
}

int orc_codec_plan(const char* method, double ratio, const kvt_kv_shape* shape, kvt_codec_cfg* out) {
  if (!method || !shape || !out) return orc_fail(KVT_EINVAL, "null argument");
  if (!(ratio > 0.0) || ratio > 1.0) return orc_fail(KVT_EVALIDATION, "codec ratio must be in (0, 1]");
  if (shape->D != D_HEAD || shape->T <= 0 || shape->L <= 0 || shape->H <= 0)
    return orc_fail(KVT_EINVAL, "unsupported KV shape");
  memset(out, 0, sizeof *out);
  const char* dash = strstr(method, "-q");
  size_t n = dash ? (size_t)(dash - method) : strlen(method);
  int bits = 16;
  if (dash) {
    bits = atoi(dash + 2);
    if (bits != 2 && bits != 4 && bits != 8) return orc_fail(KVT_EVALIDATION, "unsupported bit width in %s", method);
  }
  if (n == 5 && strncmp(method, "knorm", 5) == 0) out->scorer = KVT_SCORER_KNORM;
  else if (n == 7 && strncmp(method, "keydiff", 7) == 0) out->scorer = KVT_SCORER_KEYDIFF;
  else if (n == 6 && strncmp(method, "snapkv", 6) == 0) out->scorer = KVT_SCORER_SNAPKV;
  else return orc_fail(KVT_EVALIDATION, "unknown codec method %s", method);
  /* smallest bit width >= the method's that can hold `ratio` */
  static const int widths[4] = {2, 4, 8, 16};
  int w = 0;
  while (widths[w] < bits) ++w;
  while (widths[w] < 16 && ratio > eff_bytes(widths[w])) ++w;
  out->bits = widths[w];
  const double keep = ratio / eff_bytes(out->bits);
  long long k = (long long)floor(keep * (double)shape->T + 0.5);
  if (k < 1) k = 1;
  if (k > shape->T) k = shape->T;
  out->window = shape->T < 32 ? shape->T : 32;
  out->q_heads = 4;
  out->pool = 7;
  out->q_seed = 0x5eed5eedull;
  if (out->scorer == KVT_SCORER_SNAPKV && k < out->window) k = out->window;
  out->keep = (int32_t)k;
  return KVT_OK;
}

static int64_t al256(int64_t x) { return (x + 255) & ~(int64_t)255; }

int orc_blob_layout(const kvt_kv_shape* s, const kvt_codec_cfg* c, kvt_blob_map* o) {
  const int64_t S = (int64_t)s->L * s->H, k = c->keep, D = s->D;
  memset(o, 0, sizeof *o);
  if (k == s->T && c->bits == 16) { /* identity: the source KV is the compressed chunk */
    o->identity = 1;
    return KVT_OK;
  }
  int64_t off = 0;
  o->idx_off = off;
  o->idx_bytes = 4 * S * k;
  off = al256(off + o->idx_bytes);
  if (c->bits == 16) {
    o->kcode_off = off;
    o->kcode_bytes = 2 * S * k * D;
    off = al256(off + o->kcode_bytes);
    o->vcode_off = off;
    o->vcode_bytes = o->kcode_bytes;
    off = al256(off + o->vcode_bytes);
  } else {
    const int64_t wpr = D * c->bits / 32, ng = (k + KVT_QGROUP - 1) / KVT_QGROUP;
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
  return KVT_OK;
}

/* ------------------------------------------------------------ synthetic KV */

static uint64_t mix64(uint64_t z) { /* splitmix64 finaliser */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* bf16 bits of element `idx` of stream (seed, ctx): random sign, 7-bit
 * mantissa, exponent in [2^-3, 2^1), x8 on outlier channels (d % 16 == 3)
 * of keys and queries. Integer-only, so CPU and GPU agree exactly. */
static uint16_t synth_bf16(uint64_t seed, uint64_t ctx, uint64_t idx, int outlier) {
  uint64_t z = mix64(seed * 0x9e3779b97f4a7c15ull + ctx * 0xc2b2ae3d27d4eb4full + idx * 0x9e3779b97f4a7c15ull);
  uint32_t sign = (uint32_t)(z & 1u), mant = (uint32_t)((z >> 1) & 0x7fu);
  uint32_t e = 124u + (uint32_t)((z >> 8) & 3u) + (outlier ? 3u : 0u);
  return (uint16_t)((sign << 15) | (e << 7) | mant);
}

int orc_kv_generate(kvt_handle* h, const kvt_kv_shape* s, uint64_t seed, uint64_t ctx, uint16_t* k, uint16_t* v) {
  (void)h;
  const uint64_t n = (uint64_t)s->L * s->H * s->T * s->D;
  for (uint64_t i = 0; i < n; ++i) {
    const int d = (int)(i % (uint64_t)s->D);
    if (k) k[i] = synth_bf16(seed, ctx, i, d % 16 == 3);
    if (v) v[i] = synth_bf16(seed, ctx, n + i, 0);
  }
  return KVT_OK;
}

/* snapkv window query q[l][hq][w][d]: the caller's (bf16 [L][H*G][W][D]) or
 * the synthetic stream (q_seed, 0x51) */
static uint16_t synth_q(const kvt_kv_shape* s, const kvt_codec_cfg* c, int l, int hq, int w, int d);
static uint16_t window_q(const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* q, int l, int hq, int w,
                         int d) {
  if (!q) return synth_q(s, c, l, hq, w, d);
  const uint64_t Hq = (uint64_t)s->H * c->q_heads;
  return q[(((uint64_t)l * Hq + (uint64_t)hq) * (uint64_t)c->window + (uint64_t)w) * D_HEAD + (uint64_t)d];
}
static uint16_t synth_q(const kvt_kv_shape* s, const kvt_codec_cfg* c, int l, int hq, int w, int d) {
  const uint64_t Hq = (uint64_t)s->H * c->q_heads;
  const uint64_t idx = (((uint64_t)l * Hq + (uint64_t)hq) * (uint64_t)c->window + (uint64_t)w) * D_HEAD + (uint64_t)d;
  return synth_bf16(c->q_seed, 0x51ull, idx, d % 16 == 3);
}

/* ------------------------------------------------------------ parallel for */

typedef struct {
  void (*fn)(void*, int64_t);
  void* arg;
  int64_t n, next;
  pthread_mutex_t mu;
} pfor_t;

static void* pfor_worker(void* p) {
  pfor_t* P = (pfor_t*)p;
  for (;;) {
    pthread_mutex_lock(&P->mu);
    int64_t i = P->next++;
    pthread_mutex_unlock(&P->mu);
    if (i >= P->n) break;
    P->fn(P->arg, i);
  }
  return NULL;
}

static int orc_threads(void) {
  const char* e = getenv("ORC_THREADS");
  int n = e ? atoi(e) : (int)sysconf(_SC_NPROCESSORS_ONLN);
  return n < 1 ? 1 : (n > 256 ? 256 : n);
}

static void parallel_for(int64_t n, void (*fn)(void*, int64_t), void* arg) {
  int nt = orc_threads();
  if (nt > n) nt = (int)n;
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) fn(arg, i);
    return;
  }
  pfor_t P = {fn, arg, n, 0, PTHREAD_MUTEX_INITIALIZER};
  pthread_t th[256];
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, pfor_worker, &P);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

int orc_parallel_threads(void) { return orc_threads(); }

/* ------------------------------------------------------------------ scores */

/* canonical fp32 dot product of two 128-channel rows:
 * 16 chunks of 8 consecutive channels; inside a chunk an even-channel and an
 * odd-channel fmaf chain (channel order), chunk sum = even + odd; then a
 * butterfly over the 16 chunk sums with strides 8, 4, 2, 1. Every step is
 * one IEEE single operation, so the CUDA half-warp (one chunk per lane,
 * packed fp32x2 FMAs, xor shuffles) reproduces it bit for bit. */
static float row_dot(const float* x, const float* y) {
  float p[NCHUNK];
  for (int j = 0; j < NCHUNK; ++j) {
    float e = 0.0f, o = 0.0f;
    for (int q = 0; q < 4; ++q) {
      e = fmaf(x[8 * j + 2 * q], y[8 * j + 2 * q], e);
      o = fmaf(x[8 * j + 2 * q + 1], y[8 * j + 2 * q + 1], o);
    }
    p[j] = e + o;
  }
  for (int off = 8; off > 0; off >>= 1) {
    float q[NCHUNK];
    for (int j = 0; j < NCHUNK; ++j) q[j] = p[j] + p[j ^ off];
    memcpy(p, q, sizeof p);
  }
  return p[0];
}

static void row_f32(const uint16_t* x, float* out) {
  for (int d = 0; d < D_HEAD; ++d) out[d] = bf2f(x[d]);
}

typedef struct {
  const kvt_kv_shape* s;
  const kvt_codec_cfg* c;
  const uint16_t* k;
  const uint16_t* q; /* snapkv window queries or NULL */
  float* scores;
} score_job_t;

/* knorm: squared L2 norm of every key, larger = keep;
 * KVT_CODEC_KNORM_KEEP_LOW negates it (low norms kept, the cited knorm paper) */
static void knorm_slice(void* a, int64_t sl) {
  score_job_t* J = (score_job_t*)a;
  const int T = J->s->T;
  const float sign = (J->c->flags & KVT_CODEC_KNORM_KEEP_LOW) ? -1.0f : 1.0f;
  const uint16_t* K = J->k + (size_t)sl * T * D_HEAD;
  float x[D_HEAD];
  for (int t = 0; t < T; ++t) {
    row_f32(K + (size_t)t * D_HEAD, x);
    J->scores[(size_t)sl * T + t] = sign * row_dot(x, x);
  }
}

#define KD_FX 2097152.0f  /* 2^21: fixed-point scale of the unit directions */
#define KD_MIN_N2 0x1p-100f /* 2^-100: rows with a smaller squared norm count as zero */

/* inverse norm of a row from its squared norm: 1 / sqrt(n2), two correctly
 * rounded single ops; 0 for (near-)zero rows */
static float kd_inv(float n2) {
  if (!(n2 >= KD_MIN_N2)) return 0.0f;
  const float s = sqrtf(n2);
  return 1.0f / s;
}

/* keydiff: minus the cosine similarity of each key to the
 * sum of all unit keys of its (layer, head). The sum is exact: every unit
 * component is rounded to a 2^-21 fixed-point integer (rint of one fp32
 * product, |value| <= 2^21 + 1) and summed in int64. */
static void keydiff_slice(void* a, int64_t sl) {
  score_job_t* J = (score_job_t*)a;
  const int T = J->s->T;
  const uint16_t* K = J->k + (size_t)sl * T * D_HEAD;
  int64_t S[D_HEAD];
  memset(S, 0, sizeof S);
  float* inv = (float*)malloc(sizeof(float) * (size_t)T);
  float x[D_HEAD];
  for (int t = 0; t < T; ++t) {
    row_f32(K + (size_t)t * D_HEAD, x);
    inv[t] = kd_inv(row_dot(x, x));
    const float c = inv[t] * KD_FX;
    /* rint of the exact product x * c (one fused rounding: fma with 1.5 * 2^23) */
    for (int d = 0; d < D_HEAD; ++d) S[d] += (int64_t)(fmaf(x[d], c, 12582912.0f) - 12582912.0f);
  }
  float sd[D_HEAD];
  for (int d = 0; d < D_HEAD; ++d) sd[d] = (float)S[d] * (1.0f / KD_FX);
  for (int t = 0; t < T; ++t) {
    row_f32(K + (size_t)t * D_HEAD, x);
    J->scores[(size_t)sl * T + t] = -(row_dot(x, sd) * inv[t]); /* drop high similarity */
  }
  free(inv);
}

/* snapkv, exact-integer formulation v4.
 * Window queries quantised to int8 per row, prefix keys to int8 per
 * 16-token group, so every logit is an exact int8 dot product I_rt times
 * a per-(group, row) fp32 factor a (log2 units). Softmax over the prefix
 * per query row uses a per-(row, 32-token block) integer shift M_br =
 * ceil(max_block y): E_rt = round(2^7 * 2^(y_rt - M_br)), an 8-bit value,
 * by a fixed degree-2 fp32 FMA polynomial; the row sum and the vote weights
 * rescale blocks by exact integer shifts; votes (sum over rows of
 * probabilities, 2^37 fixed point: integer dot products of 8-bit E with
 * 30-bit weights, which the GPU computes on the integer tensor cores) are
 * max-pooled. Only IEEE single ops with a fixed association and integer
 * arithmetic appear, so the CUDA path matches it bit for bit. */
#define SNAP_C0 0.12751743082459868f /* log2(e) / sqrt(128) */
#define SNAP_E0 0x1.ffec2ep+6f        /* 2^7 * 2^f on [-1/2, 1/2], degree 2 */
#define SNAP_E1 0x1.683ef2p+6f
#define SNAP_E2 0x1.f22ab4p+4f
#define SNAP_LSH 24                   /* block sums scaled by 2^24 in the row sum */
#define SNAP_VOTE_SCALE 0x1p-37f      /* vote = 2^37 x sum of probabilities */
#define SNAP_BLK 32   /* tokens per softmax shift block */
#define SNAP_KGRP 16  /* tokens per K int8 scale (spec v4) */
#define SNAP_AMAX 0.25f /* cap of the logit factor a (v4): keeps -M - 12582912 a exact */

static uint32_t f2u(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
static float u2f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* int8 quantisation of n values with one absmax/127 scale: returns the scale */
static float quant_i8(const float* x, int n, int8_t* q) {
  float a = 0.0f;
  for (int d = 0; d < n; ++d) {
    const float v = fabsf(x[d]);
    a = v > a ? v : a;
  }
  if (a == 0.0f) {
    memset(q, 0, (size_t)n);
    return 0.0f;
  }
  const float inv = 127.0f / a;
  for (int d = 0; d < n; ++d) { /* rint of the exact product x * inv, clamped to +-127 */
    float r = fmaf(x[d], inv, 12582912.0f) - 12582912.0f;
    r = r > 127.0f ? 127.0f : (r < -127.0f ? -127.0f : r);
    q[d] = (int8_t)r;
  }
  return a / 127.0f;
}

/* E(d) = round(2^7 * 2^max(d, -16)) with the fixed polynomial above:
 * n = rint(d), f = d - n, p = poly(f), x = p * 2^n (exponent add), rint(x);
 * 0 <= E <= 128 for d <= 0. */
static uint32_t snap_exp_u8(float d) {
  const float dc = d > -16.0f ? d : -16.0f;
  const float t = dc + 12582912.0f;
  const float n = t - 12582912.0f;
  const float f = dc - n;
  float p = fmaf(SNAP_E2, f, SNAP_E1);
  p = fmaf(p, f, SNAP_E0);
  const float x = u2f(f2u(p) + (f2u(t) << 23));
  return f2u(x + 8388608.0f) - 0x4B000000u;
}

static void snapkv_slice(void* a, int64_t sl) {
  score_job_t* J = (score_job_t*)a;
  const kvt_kv_shape* s = J->s;
  const kvt_codec_cfg* c = J->c;
  const int T = s->T, W = c->window, G = c->q_heads, P = T - W, R = W * G;
  const int l = (int)(sl / s->H), h = (int)(sl % s->H);
  const uint16_t* K = J->k + (size_t)sl * T * D_HEAD;
  float* out = J->scores + (size_t)sl * T;
  for (int t = P > 0 ? P : 0; t < T; ++t) out[t] = INFINITY; /* window always kept */
  if (P <= 0) return;
  const int ngrp = (P + SNAP_KGRP - 1) / SNAP_KGRP, nblk = (P + SNAP_BLK - 1) / SNAP_BLK;
  int8_t* q8 = (int8_t*)malloc((size_t)R * D_HEAD);
  float* sig = (float*)malloc(sizeof(float) * (size_t)R);
  float row[D_HEAD];
  for (int g = 0; g < G; ++g)
    for (int w = 0; w < W; ++w) {
      const int r = g * W + w;
      for (int d = 0; d < D_HEAD; ++d) row[d] = bf2f(window_q(s, c, J->q, l, h * G + g, w, d));
      sig[r] = quant_i8(row, D_HEAD, q8 + (size_t)r * D_HEAD);
    }
  /* K: one int8 scale per 16-token group of the prefix (v4) */
  int8_t* k8 = (int8_t*)malloc((size_t)P * D_HEAD);
  float* tau = (float*)malloc(sizeof(float) * (size_t)ngrp);
  float* tile = (float*)malloc(sizeof(float) * SNAP_KGRP * D_HEAD);
  for (int j = 0; j < ngrp; ++j) {
    const int t0 = j * SNAP_KGRP, n = (P - t0 < SNAP_KGRP ? P - t0 : SNAP_KGRP);
    for (int i = 0; i < n * D_HEAD; ++i) tile[i] = bf2f(K[(size_t)t0 * D_HEAD + i]);
    tau[j] = quant_i8(tile, n * D_HEAD, k8 + (size_t)t0 * D_HEAD);
  }
  uint8_t* E = (uint8_t*)malloc((size_t)R * P);
  int32_t* Mb = (int32_t*)malloc(sizeof(int32_t) * (size_t)R * nblk);
  uint32_t* Lb = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)R * nblk);
  uint32_t* Wr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)R * nblk);
  int32_t* I = (int32_t*)malloc(sizeof(int32_t) * SNAP_BLK);
  for (int r = 0; r < R; ++r) {
    const int8_t* qr = q8 + (size_t)r * D_HEAD;
    for (int b = 0; b < nblk; ++b) {
      const int t0 = b * SNAP_BLK, n = (P - t0 < SNAP_BLK ? P - t0 : SNAP_BLK);
      /* log2 units per unit of I for each token's 16-group, capped at 1/4
       * and with the low 2 mantissa bits cleared: then 12582912 * a and
       * -M - 12582912 * a are exact (|M| <= 2^21 a), and the fma below is the
       * single correctly rounded value of I * a - M. (A factor of 1/4 log2
       * units per unit of I already makes the softmax one-hot; without the
       * cap the offset rounds and E could exceed 8 bits.) */
      float a_t[SNAP_BLK];
      float ymax = -INFINITY;
      for (int i = 0; i < n; ++i) {
        int32_t acc = 0;
        const int8_t* kt = k8 + (size_t)(t0 + i) * D_HEAD;
        for (int d = 0; d < D_HEAD; ++d) acc += (int32_t)qr[d] * (int32_t)kt[d];
        I[i] = acc;
        const float araw = (tau[(t0 + i) / SNAP_KGRP] * sig[r]) * SNAP_C0;
        a_t[i] = u2f(f2u(araw < SNAP_AMAX ? araw : SNAP_AMAX) & ~3u);
        const float y = (float)acc * a_t[i];
        ymax = y > ymax ? y : ymax;
      }
      const int32_t M = (int32_t)ceilf(ymax); /* ceil of the block's largest fl(I a) */
      uint32_t L = 0;
      for (int i = 0; i < n; ++i) {
        const float X = u2f((uint32_t)(I[i] + 0x4B400000));
        const float cb = (float)(-M) - 12582912.0f * a_t[i];
        const uint32_t e = snap_exp_u8(fmaf(X, a_t[i], cb));
        E[(size_t)r * P + t0 + i] = (uint8_t)e;
        L += e;
      }
      Mb[(size_t)r * nblk + b] = M;
      Lb[(size_t)r * nblk + b] = L;
    }
    int32_t m = INT32_MIN;
    for (int b = 0; b < nblk; ++b) m = Mb[(size_t)r * nblk + b] > m ? Mb[(size_t)r * nblk + b] : m;
    uint64_t Lr = 0;
    for (int b = 0; b < nblk; ++b) {
      const int sh = m - Mb[(size_t)r * nblk + b];
      if (sh < 64) Lr += ((uint64_t)Lb[(size_t)r * nblk + b] << SNAP_LSH) >> sh;
    }
    const uint64_t Wt = Lr ? (1ull << 61) / Lr : 0;
    for (int b = 0; b < nblk; ++b) {
      const int sh = m - Mb[(size_t)r * nblk + b];
      Wr[(size_t)r * nblk + b] = sh < 64 ? (uint32_t)(Wt >> sh) : 0u;
    }
  }
  uint64_t* vote = (uint64_t*)calloc((size_t)P, sizeof(uint64_t));
  for (int r = 0; r < R; ++r)
    for (int t = 0; t < P; ++t)
      vote[t] += (uint64_t)E[(size_t)r * P + t] * Wr[(size_t)r * nblk + t / SNAP_BLK];
  const int half = c->pool / 2;
  for (int t = 0; t < P; ++t) {
    uint64_t m = vote[t];
    for (int j = t - half; j <= t + half; ++j)
      if (j >= 0 && j < P && vote[j] > m) m = vote[j];
    out[t] = (float)m * SNAP_VOTE_SCALE;
  }
  free(q8);
  free(sig);
  free(k8);
  free(tau);
  free(tile);
  free(E);
  free(Mb);
  free(Lb);
  free(Wr);
  free(I);
  free(vote);
}

int orc_token_scores(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k,
                     const uint16_t* q, float* scores) {
  (void)h;
  if (s->D != D_HEAD) return orc_fail(KVT_EINVAL, "D must be 128");
  score_job_t J = {s, c, k, q, scores};
  const int64_t S = (int64_t)s->L * s->H;
  switch (c->scorer) {
    case KVT_SCORER_KNORM: parallel_for(S, knorm_slice, &J); break;
    case KVT_SCORER_KEYDIFF: parallel_for(S, keydiff_slice, &J); break;
    case KVT_SCORER_SNAPKV: parallel_for(S, snapkv_slice, &J); break;
    default: return orc_fail(KVT_EINVAL, "unknown scorer");
  }
  return KVT_OK;
}

/* ------------------------------------------------------------------- top-k */

static uint32_t score_key(float f) { /* larger float -> larger key; -0 == +0 */
  if (f == 0.0f) f = 0.0f;
  uint32_t x;
  memcpy(&x, &f, 4);
  return (x & 0x80000000u) ? ~x : (x | 0x80000000u);
}

typedef struct {
  const kvt_kv_shape* s;
  const kvt_codec_cfg* c;
  const float* scores;
  int32_t* idx;
} topk_job_t;

static int cmp_u32_desc(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x > y ? -1 : (x < y ? 1 : 0);
}

static void topk_slice(void* a, int64_t sl) {
  topk_job_t* J = (topk_job_t*)a;
  const int T = J->s->T, k = J->c->keep;
  const float* sc = J->scores + (size_t)sl * T;
  uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T);
  for (int t = 0; t < T; ++t) keys[t] = score_key(sc[t]);
  uint32_t* sorted = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T);
  memcpy(sorted, keys, sizeof(uint32_t) * (size_t)T);
  qsort(sorted, (size_t)T, sizeof(uint32_t), cmp_u32_desc);
  const uint32_t kth = sorted[k - 1];
  int n_above = 0;
  for (int t = 0; t < T; ++t) n_above += keys[t] > kth;
  int ties_left = k - n_above, o = 0;
  int32_t* out = J->idx + (size_t)sl * k;
  for (int t = 0; t < T; ++t) { /* ascending; ties at the threshold -> lower index */
    if (keys[t] > kth) out[o++] = t;
    else if (keys[t] == kth && ties_left > 0) {
      out[o++] = t;
      --ties_left;
    }
  }
  free(keys);
  free(sorted);
}

int orc_topk(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const float* scores, int32_t* idx) {
  (void)h;
  if (c->keep < 1 || c->keep > s->T) return orc_fail(KVT_EINVAL, "keep out of range");
  topk_job_t J = {s, c, scores, idx};
  parallel_for((int64_t)s->L * s->H, topk_slice, &J);
  return KVT_OK;
}

/* -------------------------------------------------------------- quantise */

typedef struct {
  float sf, zf, inv;
  uint16_t s16, z16;
} qparam_t;

/* asymmetric min/max group parameters, fp16 scale + zero */
static qparam_t make_param(float mn, float mx, int bits) {
  qparam_t p;
  const float levels = (float)((1 << bits) - 1);
  mn = mn + 0.0f; /* -0 -> +0: independent of which zero the min/max scan kept */
  mx = mx + 0.0f;
  const float scale = (mx - mn) / levels;
  p.s16 = f2h(scale);
  p.z16 = f2h(mn);
  p.sf = h2f(p.s16);
  p.zf = h2f(p.z16);
  p.inv = p.sf > 0.0f ? 1.0f / p.sf : 0.0f;
  return p;
}

/* code = clamp(rint(exact((x - z) * inv)), 0, 2^b - 1): the difference is
 * one fp32 op, the product is exact (double) and rounded once, ties to even */
static uint32_t quant(float x, const qparam_t* p, int bits) {
  const double y = (double)(x - p->zf) * (double)p->inv;
  double r = nearbyint(y);
  const double hi = (double)((1 << bits) - 1);
  if (!(r >= 0.0)) r = 0.0;
  if (r > hi) r = hi;
  return (uint32_t)r;
}

static float dequant(uint32_t code, float sf, float zf) {
  const float a = (float)code * sf;
  return a + zf;
}

typedef struct {
  const kvt_kv_shape* s;
  const kvt_codec_cfg* c;
  const uint16_t *k, *v;
  const int32_t* idx;
  uint8_t* blob;
  kvt_blob_map map;
} pack_job_t;

static void pack_slice(void* a, int64_t sl) {
  pack_job_t* J = (pack_job_t*)a;
  const int T = J->s->T, k = J->c->keep, bits = J->c->bits;
  const uint16_t* K = J->k + (size_t)sl * T * D_HEAD;
  const uint16_t* V = J->v + (size_t)sl * T * D_HEAD;
  const int32_t* ix = J->idx + (size_t)sl * k;
  int32_t* oidx = (int32_t*)(J->blob + J->map.idx_off) + (size_t)sl * k;
  memcpy(oidx, ix, sizeof(int32_t) * (size_t)k);
  if (bits == 16) {
    uint16_t* ko = (uint16_t*)(J->blob + J->map.kcode_off) + (size_t)sl * k * D_HEAD;
    uint16_t* vo = (uint16_t*)(J->blob + J->map.vcode_off) + (size_t)sl * k * D_HEAD;
    for (int j = 0; j < k; ++j) {
      memcpy(ko + (size_t)j * D_HEAD, K + (size_t)ix[j] * D_HEAD, 2 * D_HEAD);
      memcpy(vo + (size_t)j * D_HEAD, V + (size_t)ix[j] * D_HEAD, 2 * D_HEAD);
    }
    return;
  }
  const int wpr = D_HEAD * bits / 32, per = 32 / bits, ng = (k + KVT_QGROUP - 1) / KVT_QGROUP;
  uint32_t* kc = (uint32_t*)(J->blob + J->map.kcode_off) + (size_t)sl * k * wpr;
  uint32_t* vc = (uint32_t*)(J->blob + J->map.vcode_off) + (size_t)sl * k * wpr;
  uint16_t* ks = (uint16_t*)(J->blob + J->map.kscale_off) + (size_t)sl * ng * D_HEAD;
  uint16_t* kz = (uint16_t*)(J->blob + J->map.kzero_off) + (size_t)sl * ng * D_HEAD;
  uint16_t* vs = (uint16_t*)(J->blob + J->map.vscale_off) + (size_t)sl * k;
  uint16_t* vz = (uint16_t*)(J->blob + J->map.vzero_off) + (size_t)sl * k;
  /* K: per channel over groups of 128 kept tokens */
  for (int g = 0; g < ng; ++g) {
    const int j0 = g * KVT_QGROUP, j1 = j0 + KVT_QGROUP < k ? j0 + KVT_QGROUP : k;
    for (int d = 0; d < D_HEAD; ++d) {
      float mn = bf2f(K[(size_t)ix[j0] * D_HEAD + d]), mx = mn;
      for (int j = j0 + 1; j < j1; ++j) {
        const float x = bf2f(K[(size_t)ix[j] * D_HEAD + d]);
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
      }
      const qparam_t p = make_param(mn, mx, bits);
      ks[(size_t)g * D_HEAD + d] = p.s16;
      kz[(size_t)g * D_HEAD + d] = p.z16;
      for (int j = j0; j < j1; ++j) {
        const uint32_t code = quant(bf2f(K[(size_t)ix[j] * D_HEAD + d]), &p, bits);
        kc[(size_t)j * wpr + d / per] |= code << (bits * (d % per));
      }
    }
  }
  /* V: per token over its 128 channels */
  for (int j = 0; j < k; ++j) {
    const uint16_t* row = V + (size_t)ix[j] * D_HEAD;
    float mn = bf2f(row[0]), mx = mn;
    for (int d = 1; d < D_HEAD; ++d) {
      const float x = bf2f(row[d]);
      mn = x < mn ? x : mn;
      mx = x > mx ? x : mx;
    }
    const qparam_t p = make_param(mn, mx, bits);
    vs[j] = p.s16;
    vz[j] = p.z16;
    for (int d = 0; d < D_HEAD; ++d) vc[(size_t)j * wpr + d / per] |= quant(bf2f(row[d]), &p, bits) << (bits * (d % per));
  }
}

int orc_pack(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k, const uint16_t* v,
             const int32_t* idx, void* blob) {
  (void)h;
  pack_job_t J;
  J.s = s;
  J.c = c;
  J.k = k;
  J.v = v;
  J.idx = idx;
  J.blob = (uint8_t*)blob;
  orc_blob_layout(s, c, &J.map);
  if (J.map.identity) return KVT_OK; /* nothing to write: the source KV is the blob */
  memset(blob, 0, (size_t)J.map.total_bytes);
  parallel_for((int64_t)s->L * s->H, pack_slice, &J);
  return KVT_OK;
}

typedef struct {
  const kvt_kv_shape* s;
  const kvt_codec_cfg* c;
  const uint8_t* blob;
  uint16_t *ko, *vo;
  kvt_blob_map map;
} unpack_job_t;

static void unpack_slice(void* a, int64_t sl) {
  unpack_job_t* J = (unpack_job_t*)a;
  const int k = J->c->keep, bits = J->c->bits;
  uint16_t* ko = J->ko + (size_t)sl * k * D_HEAD;
  uint16_t* vo = J->vo + (size_t)sl * k * D_HEAD;
  if (bits == 16) {
    memcpy(ko, (const uint16_t*)(J->blob + J->map.kcode_off) + (size_t)sl * k * D_HEAD, 2 * (size_t)k * D_HEAD);
    memcpy(vo, (const uint16_t*)(J->blob + J->map.vcode_off) + (size_t)sl * k * D_HEAD, 2 * (size_t)k * D_HEAD);
    return;
  }
  const int wpr = D_HEAD * bits / 32, per = 32 / bits, ng = (k + KVT_QGROUP - 1) / KVT_QGROUP;
  const uint32_t mask = (1u << bits) - 1u;
  const uint32_t* kc = (const uint32_t*)(J->blob + J->map.kcode_off) + (size_t)sl * k * wpr;
  const uint32_t* vc = (const uint32_t*)(J->blob + J->map.vcode_off) + (size_t)sl * k * wpr;
  const uint16_t* ks = (const uint16_t*)(J->blob + J->map.kscale_off) + (size_t)sl * ng * D_HEAD;
  const uint16_t* kz = (const uint16_t*)(J->blob + J->map.kzero_off) + (size_t)sl * ng * D_HEAD;
  const uint16_t* vs = (const uint16_t*)(J->blob + J->map.vscale_off) + (size_t)sl * k;
  const uint16_t* vz = (const uint16_t*)(J->blob + J->map.vzero_off) + (size_t)sl * k;
  for (int j = 0; j < k; ++j) {
    const int g = j / KVT_QGROUP;
    const float vsf = h2f(vs[j]), vzf = h2f(vz[j]);
    for (int d = 0; d < D_HEAD; ++d) {
      const uint32_t kcode = (kc[(size_t)j * wpr + d / per] >> (bits * (d % per))) & mask;
      const uint32_t vcode = (vc[(size_t)j * wpr + d / per] >> (bits * (d % per))) & mask;
      ko[(size_t)j * D_HEAD + d] = f2bf(dequant(kcode, h2f(ks[(size_t)g * D_HEAD + d]), h2f(kz[(size_t)g * D_HEAD + d])));
      vo[(size_t)j * D_HEAD + d] = f2bf(dequant(vcode, vsf, vzf));
    }
  }
}

int orc_unpack(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const void* blob, uint16_t* k_out,
               uint16_t* v_out) {
  (void)h;
  unpack_job_t J;
  J.s = s;
  J.c = c;
  J.blob = (const uint8_t*)blob;
  J.ko = k_out;
  J.vo = v_out;
  orc_blob_layout(s, c, &J.map);
  if (J.map.identity)
    return orc_fail(KVT_EINVAL, "identity configuration: the blob aliases the source KV (kvt_blob_map.identity)");
  parallel_for((int64_t)s->L * s->H, unpack_slice, &J);
  return KVT_OK;
}

int64_t orc_compress_workspace_bytes(const kvt_kv_shape* s, const kvt_codec_cfg* c) {
  const int64_t S = (int64_t)s->L * s->H;
  return al256(4 * S * s->T) + al256(4 * S * c->keep);
}

int orc_compress(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k, const uint16_t* v,
                 const uint16_t* q, void* workspace, void* blob) {
  const int64_t S = (int64_t)s->L * s->H;
  if (c->keep == s->T && c->bits == 16) return KVT_OK; /* identity: nothing to write */
  float* scores = (float*)workspace;
  int32_t* idx = (int32_t*)((uint8_t*)workspace + al256(4 * S * s->T));
  int rc;
  if ((rc = orc_token_scores(h, s, c, k, q, scores))) return rc;
  if ((rc = orc_topk(h, s, c, scores, idx))) return rc;
  return orc_pack(h, s, c, k, v, idx, blob);
}

/* bit helpers exported for the known-answer tests */
uint16_t orc_f2h(float f) { return f2h(f); }
float orc_h2f(uint16_t h) { return h2f(h); }
uint16_t orc_f2bf(float f) { return f2bf(f); }
