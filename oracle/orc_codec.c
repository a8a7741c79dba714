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
 * bit-for-bit: FP64 sums in the canonical chunk-then-butterfly order,
 * fixed-point (2^-40) accumulation for keydiff's mean direction, fp32 IEEE
 * ops (no contraction: built with -ffp-contract=off) for quantisation,
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

/* snapkv synthetic query: q[l][hq][w][d] of stream (q_seed, 0) */
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

/* canonical FP64 sum of squares of one 128-channel row: 16 chunks of 8
 * consecutive channels summed sequentially, then a butterfly over the 16
 * chunk sums with strides 8, 4, 2, 1. */
static double row_sumsq(const uint16_t* x) {
  double p[NCHUNK];
  for (int j = 0; j < NCHUNK; ++j) {
    double acc = 0.0;
    for (int i = 0; i < 8; ++i) {
      const double v = (double)bf2f(x[8 * j + i]);
      acc = acc + v * v;
    }
    p[j] = acc;
  }
  for (int off = 8; off > 0; off >>= 1) {
    double q[NCHUNK];
    for (int j = 0; j < NCHUNK; ++j) q[j] = p[j] + p[j ^ off];
    memcpy(p, q, sizeof p);
  }
  return p[0];
}

typedef struct {
  const kvt_kv_shape* s;
  const kvt_codec_cfg* c;
  const uint16_t* k;
  float* scores;
} score_job_t;

static void knorm_slice(void* a, int64_t sl) {
  score_job_t* J = (score_job_t*)a;
  const int T = J->s->T;
  const uint16_t* K = J->k + (size_t)sl * T * D_HEAD;
  for (int t = 0; t < T; ++t) J->scores[(size_t)sl * T + t] = (float)row_sumsq(K + (size_t)t * D_HEAD);
}

#define FX_SCALE 1099511627776.0 /* 2^40 */

static void keydiff_slice(void* a, int64_t sl) {
  score_job_t* J = (score_job_t*)a;
  const int T = J->s->T;
  const uint16_t* K = J->k + (size_t)sl * T * D_HEAD;
  int64_t S[D_HEAD];
  memset(S, 0, sizeof S);
  double* inv = (double*)malloc(sizeof(double) * (size_t)T);
  for (int t = 0; t < T; ++t) {
    const double n2 = row_sumsq(K + (size_t)t * D_HEAD);
    inv[t] = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
    for (int d = 0; d < D_HEAD; ++d) {
      const double xn = (double)bf2f(K[(size_t)t * D_HEAD + d]) * inv[t];
      S[d] += llrint(xn * FX_SCALE);
    }
  }
  double Sd[D_HEAD];
  for (int d = 0; d < D_HEAD; ++d) Sd[d] = (double)S[d] * (1.0 / FX_SCALE);
  for (int t = 0; t < T; ++t) {
    double p[NCHUNK];
    for (int j = 0; j < NCHUNK; ++j) {
      double acc = 0.0;
      for (int i = 0; i < 8; ++i) {
        const int d = 8 * j + i;
        const double xn = (double)bf2f(K[(size_t)t * D_HEAD + d]) * inv[t];
        acc = acc + xn * Sd[d];
      }
      p[j] = acc;
    }
    for (int off = 8; off > 0; off >>= 1) {
      double q[NCHUNK];
      for (int j = 0; j < NCHUNK; ++j) q[j] = p[j] + p[j ^ off];
      memcpy(p, q, sizeof p);
    }
    J->scores[(size_t)sl * T + t] = (float)(-p[0]); /* drop high similarity */
  }
  free(inv);
}

/* snapkv, exact-integer formulation: the
 * window queries and the prefix keys are quantised to int8 per row (absmax /
 * 127), so every logit is an exact integer dot product times two fp32
 * scales; exp2 is a fixed mul/add polynomial, and every sum is an integer.
 * Only IEEE single ops with a fixed association appear, so the CUDA path
 * (integer tensor cores) reproduces it bit for bit. */
#define SNAP_C0 0.12751743082459868f /* log2(e) / sqrt(128) */
#define SNAP_P0 1.535336188319500E-4f /* 2^f on [-1/2, 1/2] (Cephes exp2f) */
#define SNAP_P1 1.339887440266574E-3f
#define SNAP_P2 9.618437357674640E-3f
#define SNAP_P3 5.550332471162809E-2f
#define SNAP_P4 2.402264791363012E-1f
#define SNAP_P5 6.931472028550421E-1f

/* int8 row quantisation: returns the scale absmax/127, writes the codes */
static float quant_row_i8(const float* x, int8_t* q) {
  float a = 0.0f;
  for (int d = 0; d < D_HEAD; ++d) {
    const float v = fabsf(x[d]);
    a = v > a ? v : a;
  }
  if (a == 0.0f) {
    memset(q, 0, D_HEAD);
    return 0.0f;
  }
  const float inv = 127.0f / a;
  for (int d = 0; d < D_HEAD; ++d) {
    float r = nearbyintf(x[d] * inv);
    r = r > 127.0f ? 127.0f : (r < -127.0f ? -127.0f : r);
    q[d] = (int8_t)r;
  }
  return a / 127.0f;
}

/* round(2^22 * 2^d) for d <= 0, 0 below d = -30 */
static uint32_t snap_exp_fx(float d) {
  if (d < -30.0f) return 0u;
  const float n = nearbyintf(d);
  const float f = d - n;
  float p = SNAP_P0;
  p = p * f + SNAP_P1;
  p = p * f + SNAP_P2;
  p = p * f + SNAP_P3;
  p = p * f + SNAP_P4;
  p = p * f + SNAP_P5;
  p = p * f + 1.0f;
  const float x = ldexpf(p, 22 + (int)n);
  return (uint32_t)nearbyintf(x);
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
  int8_t* q8 = (int8_t*)malloc((size_t)R * D_HEAD);
  float* cr = (float*)malloc(sizeof(float) * (size_t)R);
  float row[D_HEAD];
  for (int g = 0; g < G; ++g)
    for (int w = 0; w < W; ++w) {
      const int r = g * W + w;
      for (int d = 0; d < D_HEAD; ++d) row[d] = bf2f(synth_q(s, c, l, h * G + g, w, d));
      cr[r] = quant_row_i8(row, q8 + (size_t)r * D_HEAD) * SNAP_C0;
    }
  int8_t* k8 = (int8_t*)malloc((size_t)P * D_HEAD);
  float* tau = (float*)malloc(sizeof(float) * (size_t)P);
  for (int t = 0; t < P; ++t) {
    for (int d = 0; d < D_HEAD; ++d) row[d] = bf2f(K[(size_t)t * D_HEAD + d]);
    tau[t] = quant_row_i8(row, k8 + (size_t)t * D_HEAD);
  }
  float* y = (float*)malloc(sizeof(float) * (size_t)R * P);
  for (int r = 0; r < R; ++r)
    for (int t = 0; t < P; ++t) {
      int32_t acc = 0;
      for (int d = 0; d < D_HEAD; ++d) acc += (int32_t)q8[(size_t)r * D_HEAD + d] * (int32_t)k8[(size_t)t * D_HEAD + d];
      y[(size_t)r * P + t] = ((float)acc * tau[t]) * cr[r];
    }
  uint64_t* vote = (uint64_t*)calloc((size_t)P, sizeof(uint64_t));
  for (int r = 0; r < R; ++r) {
    const float* yr = y + (size_t)r * P;
    float m = yr[0];
    for (int t = 1; t < P; ++t) m = yr[t] > m ? yr[t] : m;
    uint64_t L = 0;
    for (int t = 0; t < P; ++t) L += snap_exp_fx(yr[t] - m);
    const uint64_t w = (1ull << 46) / L;
    for (int t = 0; t < P; ++t) vote[t] += (uint64_t)snap_exp_fx(yr[t] - m) * w;
  }
  const int half = c->pool / 2;
  for (int t = 0; t < P; ++t) {
    uint64_t m = vote[t];
    for (int j = t - half; j <= t + half; ++j)
      if (j >= 0 && j < P && vote[j] > m) m = vote[j];
    out[t] = (float)m * 1.4210854715202004e-14f; /* 2^-46 */
  }
  free(q8);
  free(cr);
  free(k8);
  free(tau);
  free(y);
  free(vote);
}

int orc_token_scores(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k, float* scores) {
  (void)h;
  if (s->D != D_HEAD) return orc_fail(KVT_EINVAL, "D must be 128");
  score_job_t J = {s, c, k, scores};
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

static uint32_t quant(float x, const qparam_t* p, int bits) {
  const float y = (x - p->zf) * p->inv;
  float r = nearbyintf(y);
  const float hi = (float)((1 << bits) - 1);
  if (!(r >= 0.0f)) r = 0.0f;
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
  parallel_for((int64_t)s->L * s->H, unpack_slice, &J);
  return KVT_OK;
}

int64_t orc_compress_workspace_bytes(const kvt_kv_shape* s, const kvt_codec_cfg* c) {
  const int64_t S = (int64_t)s->L * s->H;
  return al256(4 * S * s->T) + al256(4 * S * c->keep);
}

int orc_compress(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k, const uint16_t* v,
                 void* workspace, void* blob) {
  const int64_t S = (int64_t)s->L * s->H;
  float* scores = (float*)workspace;
  int32_t* idx = (int32_t*)((uint8_t*)workspace + al256(4 * S * s->T));
  int rc;
  if ((rc = orc_token_scores(h, s, c, k, scores))) return rc;
  if ((rc = orc_topk(h, s, c, scores, idx))) return rc;
  return orc_pack(h, s, c, k, v, idx, blob);
}

/* bit helpers exported for the known-answer tests */
uint16_t orc_f2h(float f) { return f2h(f); }
float orc_h2f(uint16_t h) { return h2f(h); }
uint16_t orc_f2bf(float f) { return f2bf(f); }
