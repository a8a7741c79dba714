/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's placement
 * hot path (scoring + least-utility-drop greedy), used by tests/ as the
 * checker of the CUDA path. Pinned against the reference library built from
 * /root/reference (oracle/_ref) and the reference's own known answers
 * (tests/test_oracle_pinned.py).
 *
 * Each function cites the reference file:line it restates. The structure is
 * deliberately the reference's own (a full rescan of every resident on every
 * overflow step, proj/src/placement.cpp:174-204), not the cached structure
 * of the CUDA path, so that the two are independent.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "orc_common.h"

static __thread char g_err[1024];

int orc_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }
int orc_abi_version(void) { return KVT_ABI_VERSION; }

struct kvt_handle {
  int unused;
};

int orc_create(int device, void* stream, kvt_handle** out) {
  (void)device;
  (void)stream;
  *out = (kvt_handle*)calloc(1, sizeof(kvt_handle));
  return *out ? KVT_OK : KVT_ENOMEM;
}

int orc_destroy(kvt_handle* h) {
  free(h);
  return KVT_OK;
}

/* ---------------------------------------------------------------- profiles */

struct kvt_pset {
  int32_t n, M;
  int64_t* orig;
  double* freq;
  int32_t* goff;
  double* grid;
  double* qual;
  uint8_t* has;
};

int orc_pset_create(kvt_handle* h, const kvt_profiles* pr, kvt_pset** out) {
  (void)h;
  if (!pr || pr->n_ctx < 0 || pr->n_methods <= 0) return orc_fail(KVT_EINVAL, "bad profiles");
  kvt_pset* p = (kvt_pset*)calloc(1, sizeof(kvt_pset));
  int32_t n = pr->n_ctx, M = pr->n_methods;
  int32_t G = pr->grid_offset[n];
  p->n = n;
  p->M = M;
  p->orig = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  p->freq = (double*)malloc(sizeof(double) * (n ? n : 1));
  p->goff = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  p->grid = (double*)malloc(sizeof(double) * (G ? G : 1));
  p->qual = (double*)malloc(sizeof(double) * ((size_t)G * M + 1));
  p->has = (uint8_t*)malloc((size_t)n * M + 1);
  memcpy(p->orig, pr->original_size_bytes, sizeof(int64_t) * n);
  memcpy(p->freq, pr->frequency, sizeof(double) * n);
  memcpy(p->goff, pr->grid_offset, sizeof(int32_t) * (n + 1));
  memcpy(p->grid, pr->grid, sizeof(double) * G);
  memcpy(p->qual, pr->quality, sizeof(double) * (size_t)G * M);
  memcpy(p->has, pr->has_method, (size_t)n * M);
  for (int32_t c = 0; c < n; ++c) {
    if (p->goff[c + 1] <= p->goff[c]) {
      orc_pset_destroy(p);
      return orc_fail(KVT_EVALIDATION, "profile ratio grid is empty for context %d", c);
    }
  }
  *out = p;
  return KVT_OK;
}

/* ---- multi-GPU profile exchange (include/kvt_b200.h "record"): restated on
 * host memory so the gloo multi-process tests can run the rank logic */
typedef struct {
  int64_t orig, freq, grid, qual, goff, has, total;
} rec_layout_t;

static int64_t rec_al(int64_t x) { return (x + 255) & ~(int64_t)255; }

static rec_layout_t rec_layout(int64_t n, int64_t g, int64_t M) {
  rec_layout_t L;
  L.orig = 0;
  L.freq = L.orig + rec_al(8 * n);
  L.grid = L.freq + rec_al(8 * n);
  L.qual = L.grid + rec_al(8 * g);
  L.goff = L.qual + rec_al(8 * g * M);
  L.has = L.goff + rec_al(4 * (n + 1));
  L.total = L.has + rec_al(n * M);
  return L;
}

int64_t orc_pset_record_bytes(int32_t n_ctx, int32_t grid_len, int32_t n_methods) {
  return rec_layout(n_ctx, grid_len, n_methods).total;
}

int orc_pset_record_pack(const kvt_profiles* pr, void* record) {
  if (!pr || !record || pr->n_ctx < 0 || pr->n_methods <= 0) return orc_fail(KVT_EINVAL, "bad profiles");
  const int32_t n = pr->n_ctx, M = pr->n_methods, g = pr->grid_offset[n];
  for (int32_t c = 0; c < n; ++c) {
    if (pr->grid_offset[c + 1] <= pr->grid_offset[c])
      return orc_fail(KVT_EVALIDATION, "profile ratio grid is empty for context %d", c);
    if (pr->original_size_bytes[c] <= 0) return orc_fail(KVT_EVALIDATION, "original size must be > 0");
  }
  const rec_layout_t L = rec_layout(n, g, M);
  uint8_t* b = (uint8_t*)record;
  memset(b, 0, (size_t)L.total);
  memcpy(b + L.orig, pr->original_size_bytes, 8 * (size_t)n);
  memcpy(b + L.freq, pr->frequency, 8 * (size_t)n);
  memcpy(b + L.grid, pr->grid, 8 * (size_t)g);
  memcpy(b + L.qual, pr->quality, 8 * (size_t)g * M);
  memcpy(b + L.goff, pr->grid_offset, 4 * (size_t)(n + 1));
  memcpy(b + L.has, pr->has_method, (size_t)n * M);
  return KVT_OK;
}

int orc_pset_merge(kvt_handle* h, const void* records, int32_t world, int32_t n_ctx, int32_t grid_len,
                   int32_t n_methods, kvt_pset** out) {
  (void)h;
  if (!records || !out || world < 1 || n_ctx < 0 || grid_len < 0 || n_methods <= 0)
    return orc_fail(KVT_EINVAL, "bad merge request");
  const rec_layout_t L = rec_layout(n_ctx, grid_len, n_methods);
  const int64_t N = (int64_t)world * n_ctx, G = (int64_t)world * grid_len, M = n_methods;
  if (*out) orc_pset_destroy(*out);
  kvt_pset* p = (kvt_pset*)calloc(1, sizeof(kvt_pset));
  p->n = (int32_t)N;
  p->M = n_methods;
  p->orig = (int64_t*)malloc(8 * (size_t)(N ? N : 1));
  p->freq = (double*)malloc(8 * (size_t)(N ? N : 1));
  p->goff = (int32_t*)malloc(4 * (size_t)(N + 1));
  p->grid = (double*)malloc(8 * (size_t)(G ? G : 1));
  p->qual = (double*)malloc(8 * (size_t)(G * M + 1));
  p->has = (uint8_t*)malloc((size_t)(N * M + 1));
  for (int32_t r = 0; r < world; ++r) {
    const uint8_t* b = (const uint8_t*)records + (size_t)r * L.total;
    memcpy(p->orig + (size_t)r * n_ctx, b + L.orig, 8 * (size_t)n_ctx);
    memcpy(p->freq + (size_t)r * n_ctx, b + L.freq, 8 * (size_t)n_ctx);
    memcpy(p->grid + (size_t)r * grid_len, b + L.grid, 8 * (size_t)grid_len);
    memcpy(p->qual + (size_t)r * grid_len * M, b + L.qual, 8 * (size_t)grid_len * M);
    memcpy(p->has + (size_t)r * n_ctx * M, b + L.has, (size_t)n_ctx * M);
    const int32_t* go = (const int32_t*)(b + L.goff);
    for (int32_t i = 0; i < n_ctx; ++i) p->goff[(size_t)r * n_ctx + i] = r * grid_len + go[i];
  }
  p->goff[N] = (int32_t)G;
  *out = p;
  return KVT_OK;
}

int orc_pset_destroy(kvt_pset* p) {
  if (!p) return KVT_OK;
  free(p->orig);
  free(p->freq);
  free(p->goff);
  free(p->grid);
  free(p->qual);
  free(p->has);
  free(p);
  return KVT_OK;
}

/* ------------------------------------------------------------------ space */

typedef struct {
  int32_t M, R;
  const char* names[KVT_MAX_METHODS];
  double ovh[KVT_MAX_METHODS];
  double ratio[KVT_MAX_RATIOS];
} space_t;

static int cmp_desc(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x > y ? -1 : (x < y ? 1 : 0);
}

/* CandidateSpace ctor proj/src/utility.cpp:21-33 and MethodSet ctor
 * proj/src/core.cpp:10-27. */
static int resolve_space(const kvt_space* sp, space_t* s) {
  if (!sp) return orc_fail(KVT_EINVAL, "null space");
  if (sp->n_methods <= 0) return orc_fail(KVT_EVALIDATION, "method set must not be empty");
  if (sp->n_methods > KVT_MAX_METHODS) return orc_fail(KVT_EINVAL, "too many methods");
  if (sp->n_ratios <= 0) return orc_fail(KVT_EVALIDATION, "candidate ratio grid must not be empty");
  if (sp->n_ratios > KVT_MAX_RATIOS) return orc_fail(KVT_EINVAL, "too many ratios");
  s->M = sp->n_methods;
  for (int m = 0; m < s->M; ++m) {
    const char* nm = sp->method_names[m];
    if (!nm || !nm[0]) return orc_fail(KVT_EVALIDATION, "compression method name must not be empty");
    for (int j = 0; j < m; ++j)
      if (strcmp(s->names[j], nm) == 0)
        return orc_fail(KVT_EVALIDATION, "duplicate compression method name: %s", nm);
    if (sp->decompression_overhead[m] < 0.0)
      return orc_fail(KVT_EVALIDATION, "negative decompression overhead for method %s", nm);
    s->names[m] = nm;
    s->ovh[m] = sp->decompression_overhead[m];
  }
  double tmp[KVT_MAX_RATIOS];
  for (int r = 0; r < sp->n_ratios; ++r) {
    double v = sp->ratios[r];
    if (!(v > 0.0) || v > 1.0 || !isfinite(v))
      return orc_fail(KVT_EVALIDATION, "candidate ratio out of (0, 1]");
    tmp[r] = v;
  }
  qsort(tmp, (size_t)sp->n_ratios, sizeof(double), cmp_desc);
  s->R = 0;
  for (int r = 0; r < sp->n_ratios; ++r)
    if (s->R == 0 || tmp[r] != s->ratio[s->R - 1]) s->ratio[s->R++] = tmp[r];
  return KVT_OK;
}

/* ------------------------------------------------------------------ tiers */

typedef struct {
  int32_t T;
  kvt_tier t[KVT_MAX_TIERS];
} tiers_t;

/* validate_hierarchy proj/src/core.cpp:86-121 (stable sort by tier_id). */
static int resolve_tiers(const kvt_tier* in, int32_t n, tiers_t* o) {
  if (n <= 0) return orc_fail(KVT_EVALIDATION, "hierarchy must have at least one tier");
  if (n > KVT_MAX_TIERS) return orc_fail(KVT_EINVAL, "too many tiers");
  o->T = n;
  for (int i = 0; i < n; ++i) o->t[i] = in[i];
  for (int i = 1; i < n; ++i) { /* stable insertion sort */
    kvt_tier x = o->t[i];
    int j = i - 1;
    while (j >= 0 && o->t[j].tier_id > x.tier_id) {
      o->t[j + 1] = o->t[j];
      --j;
    }
    o->t[j + 1] = x;
  }
  for (int i = 0; i < n; ++i) {
    const kvt_tier* t = &o->t[i];
    if (i + 1 < n && o->t[i + 1].tier_id == t->tier_id)
      return orc_fail(KVT_EVALIDATION, "duplicate tier_id %d", t->tier_id);
    if (t->unlimited && i + 1 != n)
      return orc_fail(KVT_EVALIDATION,
                      "unlimited capacity is only allowed on the bottom tier (tier %d)", t->tier_id);
    if (!t->unlimited && t->capacity_bytes < 0)
      return orc_fail(KVT_EVALIDATION, "negative capacity on tier %d", t->tier_id);
    if (!(t->read_bandwidth > 0.0) || !isfinite(t->read_bandwidth))
      return orc_fail(KVT_EVALIDATION, "read bandwidth must be > 0 on tier %d", t->tier_id);
    if (t->fixed_access_latency < 0.0 || !isfinite(t->fixed_access_latency))
      return orc_fail(KVT_EVALIDATION, "fixed access latency must be >= 0 on tier %d", t->tier_id);
  }
  return KVT_OK;
}

/* ------------------------------------------------------ scalar arithmetic */

#define GRID_EPS 1e-9 /* proj/src/quality.cpp:16 */

/* compressed_size proj/src/core.cpp:72-84 */
static int csize(int64_t orig, double ratio, int64_t* out) {
  if (orig <= 0) return orc_fail(KVT_EVALIDATION, "original size must be > 0");
  if (!(ratio > 0.0) || ratio > 1.0 || !isfinite(ratio))
    return orc_fail(KVT_EVALIDATION, "compression ratio must be in (0, 1], got %g", ratio);
  const double scaled = (double)orig * ratio;
  int64_t b = (int64_t)floor(scaled + 0.5);
  *out = b > 1 ? b : 1;
  return KVT_OK;
}

/* scorable proj/src/utility.cpp:13-17 */
static int scorable(const kvt_pset* p, int32_t c, int32_t m, double ratio) {
  if (!p->has[(size_t)c * p->M + m]) return 0;
  return ratio >= p->grid[p->goff[c]] - GRID_EPS;
}

/* quality_of proj/src/quality.cpp:86-113 */
static int quality_of(const kvt_pset* p, int32_t c, int32_t m, const space_t* s, double ratio,
                      double* out) {
  if (!(ratio > 0.0) || ratio > 1.0 + GRID_EPS)
    return orc_fail(KVT_EVALIDATION, "ratio out of (0,1]: %.6g", ratio);
  if (!p->has[(size_t)c * p->M + m])
    return orc_fail(KVT_EVALIDATION, "method %s not profiled for context %d", s->names[m], c);
  const int32_t g0 = p->goff[c], len = p->goff[c + 1] - g0;
  const double* grid = p->grid + g0;
  const double* val = p->qual + (size_t)g0 * p->M + (size_t)m * len;
  if (ratio < grid[0] - GRID_EPS)
    return orc_fail(KVT_EVALIDATION, "ratio %.6g below smallest profiled ratio %.6g for context %d",
                    ratio, grid[0], c);
  const double key = ratio - GRID_EPS;
  int32_t i = 0; /* std::lower_bound: first grid[i] >= key */
  while (i < len && grid[i] < key) ++i;
  if (i >= len) i = len - 1;
  if (fabs(grid[i] - ratio) <= GRID_EPS || i == 0) {
    *out = val[i];
    return KVT_OK;
  }
  const double x0 = grid[i - 1], x1 = grid[i];
  const double y0 = val[i - 1], y1 = val[i];
  const double t = (ratio - x0) / (x1 - x0);
  *out = y0 + t * (y1 - y0);
  return KVT_OK;
}

/* load_time proj/src/utility.cpp:51-59 */
static double load_time(int64_t size, const kvt_tier* t, double ovh) {
  const double s = (double)size;
  return t->fixed_access_latency + s / t->read_bandwidth + s * ovh;
}

/* utility_score proj/src/utility.cpp:61-63 */
static double utility_score(double q, double ttft, double f, double alpha) {
  return (alpha * q - ttft) * f;
}

typedef struct {
  int32_t tier_index, tier_id, method;
  double ratio;
  int64_t size;
  double quality, ttft, frequency, utility;
} cand_t;

/* score_candidate proj/src/utility.cpp:65-79 */
static int score(const kvt_pset* p, int32_t c, int32_t m, double ratio, const tiers_t* tr,
                 int32_t ti, const space_t* s, double alpha, cand_t* o) {
  int rc;
  o->tier_index = ti;
  o->tier_id = tr->t[ti].tier_id;
  o->method = m;
  o->ratio = ratio;
  if ((rc = csize(p->orig[c], ratio, &o->size))) return rc;
  if ((rc = quality_of(p, c, m, s, ratio, &o->quality))) return rc;
  o->ttft = load_time(o->size, &tr->t[ti], s->ovh[m]);
  o->frequency = p->freq[c];
  o->utility = utility_score(o->quality, o->ttft, o->frequency, alpha);
  return KVT_OK;
}

/* candidate_preferred proj/src/utility.cpp:147-157 */
static int preferred(const cand_t* a, const cand_t* b, int rule, const space_t* s) {
  if (rule == KVT_RULE_QUALITY_FIRST && a->quality != b->quality) return a->quality > b->quality;
  if (a->utility != b->utility) return a->utility > b->utility;
  if (a->quality != b->quality) return a->quality > b->quality;
  if (a->tier_id != b->tier_id) return a->tier_id < b->tier_id;
  if (a->ratio != b->ratio) return a->ratio > b->ratio;
  return strcmp(s->names[a->method], s->names[b->method]) < 0;
}

int orc_score_candidates(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, int32_t n_tiers,
                         const kvt_space* space, const kvt_params* params, int64_t* size,
                         double* quality, uint8_t* valid, double* ttft, double* utility) {
  (void)h;
  space_t s;
  tiers_t tr;
  int rc;
  if ((rc = resolve_space(space, &s))) return rc;
  if ((rc = resolve_tiers(tiers, n_tiers, &tr))) return rc;
  if (p->M != s.M) return orc_fail(KVT_EINVAL, "profile set built for %d methods, space has %d", p->M, s.M);
  const int32_t T = tr.T, M = s.M, R = s.R;
  for (int32_t c = 0; c < p->n; ++c) {
    for (int32_t r = 0; r < R; ++r) {
      int64_t sz;
      if ((rc = csize(p->orig[c], s.ratio[r], &sz))) return rc;
      if (size) size[(size_t)c * R + r] = sz;
    }
    /* all_candidates order tier -> method -> ratio, proj/src/utility.cpp:129-145 */
    for (int32_t t = 0; t < T; ++t)
      for (int32_t m = 0; m < M; ++m)
        for (int32_t r = 0; r < R; ++r) {
          const size_t qi = ((size_t)c * M + m) * R + r;
          const size_t ui = (((size_t)c * T + t) * M + m) * R + r;
          const int ok = scorable(p, c, m, s.ratio[r]);
          if (t == 0 && valid) valid[qi] = (uint8_t)ok;
          cand_t cd;
          if (!ok) {
            if (t == 0 && quality) quality[qi] = 0.0;
            if (ttft) ttft[ui] = 0.0;
            if (utility) utility[ui] = 0.0;
            continue;
          }
          if ((rc = score(p, c, m, s.ratio[r], &tr, t, &s, params->alpha, &cd))) return rc;
          if (t == 0 && quality) quality[qi] = cd.quality;
          if (ttft) ttft[ui] = cd.ttft;
          if (utility) utility[ui] = cd.utility;
        }
  }
  return KVT_OK;
}

/* best_config proj/src/utility.cpp:159-172 for one context */
static int best_one(const kvt_pset* p, int32_t c, const tiers_t* tr, const space_t* s,
                    double alpha, int rule, cand_t* best, int32_t* best_r) {
  int found = 0, rc;
  for (int32_t t = 0; t < tr->T; ++t)
    for (int32_t m = 0; m < s->M; ++m)
      for (int32_t r = 0; r < s->R; ++r) {
        if (!scorable(p, c, m, s->ratio[r])) continue;
        cand_t cd;
        if ((rc = score(p, c, m, s->ratio[r], tr, t, s, alpha, &cd))) return rc;
        if (!found || preferred(&cd, best, rule, s)) {
          *best = cd;
          *best_r = r;
          found = 1;
        }
      }
  if (!found) return orc_fail(KVT_EVALIDATION, "no scorable configuration for context %d", c);
  return KVT_OK;
}

int orc_best_config(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, int32_t n_tiers,
                    const kvt_space* space, const kvt_params* params, int32_t rule, kvt_best* out) {
  (void)h;
  space_t s;
  tiers_t tr;
  int rc;
  if ((rc = resolve_space(space, &s))) return rc;
  if ((rc = resolve_tiers(tiers, n_tiers, &tr))) return rc;
  if (p->M != s.M) return orc_fail(KVT_EINVAL, "method count mismatch");
  for (int32_t c = 0; c < p->n; ++c) {
    cand_t b;
    int32_t br = -1;
    memset(&out[c], 0, sizeof(kvt_best));
    rc = best_one(p, c, &tr, &s, params->alpha, rule, &b, &br);
    if (rc == KVT_EVALIDATION) {
      out[c].status = 1;
      continue;
    }
    if (rc) return rc;
    out[c].tier_index = b.tier_index;
    out[c].tier_id = b.tier_id;
    out[c].method = b.method;
    out[c].ratio_index = br;
    out[c].ratio = b.ratio;
    out[c].size_bytes = b.size;
    out[c].quality = b.quality;
    out[c].ttft = b.ttft;
    out[c].utility = b.utility;
  }
  return KVT_OK;
}

/* ------------------------------------------------------------------ store */

typedef struct {
  int32_t* ids; /* arrival order */
  int32_t n, cap;
} tierlist_t;

struct kvt_store {
  tiers_t tr;
  int32_t n_ctx;
  kvt_entry* e; /* per ctx; tier_index -1 = absent */
  tierlist_t* lists;
  int64_t occ[KVT_MAX_TIERS];
  int64_t seq;
  kvt_action* act;
  int64_t n_act, cap_act;
};

static void push_action(kvt_store* s, int kind, int32_t ctx, int32_t tier_id, int32_t m, double ratio) {
  if (s->n_act == s->cap_act) {
    s->cap_act = s->cap_act ? 2 * s->cap_act : 1024;
    s->act = (kvt_action*)realloc(s->act, sizeof(kvt_action) * (size_t)s->cap_act);
  }
  kvt_action* a = &s->act[s->n_act++];
  a->kind = kind;
  a->ctx = ctx;
  a->tier_id = tier_id;
  a->method = m;
  a->ratio = ratio;
}

int orc_store_create(kvt_handle* h, const kvt_tier* tiers, int32_t n_tiers, int32_t n_ctx,
                     kvt_store** out) {
  (void)h;
  kvt_store* s = (kvt_store*)calloc(1, sizeof(kvt_store));
  int rc = resolve_tiers(tiers, n_tiers, &s->tr);
  if (rc) {
    free(s);
    return rc;
  }
  s->n_ctx = n_ctx;
  s->e = (kvt_entry*)calloc((size_t)(n_ctx ? n_ctx : 1), sizeof(kvt_entry));
  for (int32_t c = 0; c < n_ctx; ++c) s->e[c].tier_index = -1;
  s->lists = (tierlist_t*)calloc((size_t)s->tr.T, sizeof(tierlist_t));
  *out = s;
  return KVT_OK;
}

int orc_store_destroy(kvt_store* s) {
  if (!s) return KVT_OK;
  for (int t = 0; t < s->tr.T; ++t) free(s->lists[t].ids);
  free(s->lists);
  free(s->e);
  free(s->act);
  free(s);
  return KVT_OK;
}

static int check_ctx(const kvt_store* s, int32_t c) {
  if (c < 0 || c >= s->n_ctx) return orc_fail(KVT_EINVAL, "context index %d out of range", c);
  return KVT_OK;
}

/* StoreState::add proj/src/placement.cpp:91-108 */
int orc_store_add(kvt_store* s, int32_t c, const kvt_entry* in) {
  int rc;
  if ((rc = check_ctx(s, c))) return rc;
  if (s->e[c].tier_index >= 0) return orc_fail(KVT_EVALIDATION, "context %d is already resident", c);
  if (in->tier_index < 0 || in->tier_index >= s->tr.T)
    return orc_fail(KVT_EVALIDATION, "unknown tier index %d", in->tier_index);
  int64_t b;
  if ((rc = csize(in->original_size_bytes, in->ratio, &b))) return rc;
  s->occ[in->tier_index] += b;
  s->e[c] = *in;
  s->e[c].seq = s->seq++;
  tierlist_t* L = &s->lists[in->tier_index];
  if (L->n == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 64;
    L->ids = (int32_t*)realloc(L->ids, sizeof(int32_t) * (size_t)L->cap);
  }
  L->ids[L->n++] = c;
  return KVT_OK;
}

/* StoreState::remove proj/src/placement.cpp:110-125 (order preserving) */
int orc_store_remove(kvt_store* s, int32_t c, kvt_entry* removed) {
  int rc;
  if ((rc = check_ctx(s, c))) return rc;
  int32_t t = s->e[c].tier_index;
  if (t < 0) return orc_fail(KVT_EVALIDATION, "context %d is not resident", c);
  tierlist_t* L = &s->lists[t];
  int32_t i = 0;
  while (i < L->n && L->ids[i] != c) ++i;
  memmove(L->ids + i, L->ids + i + 1, sizeof(int32_t) * (size_t)(L->n - i - 1));
  L->n--;
  int64_t b;
  csize(s->e[c].original_size_bytes, s->e[c].ratio, &b);
  s->occ[t] -= b;
  if (removed) *removed = s->e[c];
  s->e[c].tier_index = -1;
  return KVT_OK;
}

/* StoreState::reconfigure proj/src/placement.cpp:127-133 */
int orc_store_reconfigure(kvt_store* s, int32_t c, int32_t m, double ratio) {
  int rc;
  if ((rc = check_ctx(s, c))) return rc;
  int32_t t = s->e[c].tier_index;
  if (t < 0) return orc_fail(KVT_EVALIDATION, "context %d is not resident", c);
  int64_t b0, b1;
  csize(s->e[c].original_size_bytes, s->e[c].ratio, &b0);
  if ((rc = csize(s->e[c].original_size_bytes, ratio, &b1))) return rc;
  s->occ[t] += b1 - b0;
  s->e[c].method = m;
  s->e[c].ratio = ratio;
  return KVT_OK;
}

/* StoreState::touch proj/src/placement.cpp:135-142 */
int orc_store_touch(kvt_store* s, int32_t c, int64_t stamp) {
  int rc;
  if ((rc = check_ctx(s, c))) return rc;
  if (s->e[c].tier_index < 0) return orc_fail(KVT_EVALIDATION, "context %d is not resident", c);
  s->e[c].frequency += 1;
  s->e[c].last_access = stamp;
  return KVT_OK;
}

/* n StoreState::touch calls in order (the serve loop's hits) */
int orc_store_touch_many(kvt_store* s, const int32_t* ctx, const int64_t* stamps, int64_t n) {
  int rc;
  for (int64_t i = 0; i < n; ++i)
    if ((rc = orc_store_touch(s, ctx[i], stamps[i]))) return rc;
  return KVT_OK;
}

/* StoreState::clear proj/src/placement.cpp:144-148 */
int orc_store_clear(kvt_store* s) {
  for (int32_t c = 0; c < s->n_ctx; ++c) s->e[c].tier_index = -1;
  for (int t = 0; t < s->tr.T; ++t) {
    s->lists[t].n = 0;
    s->occ[t] = 0;
  }
  return KVT_OK;
}

int orc_store_occupancy(kvt_store* s, int64_t* occ) {
  for (int t = 0; t < s->tr.T; ++t) occ[t] = s->occ[t];
  return KVT_OK;
}

int orc_store_snapshot(kvt_store* s, kvt_entry* out) {
  memcpy(out, s->e, sizeof(kvt_entry) * (size_t)s->n_ctx);
  return KVT_OK;
}

int orc_store_actions(kvt_store* s, kvt_action* out, int64_t n) {
  if (n > s->n_act) n = s->n_act;
  memcpy(out, s->act, sizeof(kvt_action) * (size_t)n);
  return KVT_OK;
}

/* StoreState::over_capacity / first_over_capacity proj/src/placement.cpp:49-59 */
static int first_over(const kvt_store* s) {
  for (int t = 0; t < s->tr.T; ++t)
    if (!s->tr.t[t].unlimited && s->occ[t] > s->tr.t[t].capacity_bytes) return t;
  return -1;
}

/* enumerate_updates proj/src/utility.cpp:81-127; returns option count */
static int enumerate_updates(const kvt_entry* e, int32_t c, const kvt_pset* p, const tiers_t* tr,
                             const space_t* s, double alpha, cand_t* out, int* n_out) {
  int rc, n = 0;
  const int32_t cur = e->tier_index;
  int64_t cur_bytes;
  if ((rc = csize(e->original_size_bytes, e->ratio, &cur_bytes))) return rc;
  for (int32_t ti = cur; ti < tr->T; ++ti) {
    int covered = 0;
    for (int32_t m = 0; m < s->M; ++m)
      for (int32_t r = 0; r < s->R; ++r) {
        const double ratio = s->ratio[r];
        if (!scorable(p, c, m, ratio)) continue;
        if (ti == cur) {
          int64_t b;
          if ((rc = csize(e->original_size_bytes, ratio, &b))) return rc;
          if (b >= cur_bytes) continue;
        } else if (m == e->method && ratio == e->ratio) {
          covered = 1;
        }
        if ((rc = score(p, c, m, ratio, tr, ti, s, alpha, &out[n++]))) return rc;
      }
    if (ti != cur && !covered && scorable(p, c, e->method, e->ratio)) {
      if ((rc = score(p, c, e->method, e->ratio, tr, ti, s, alpha, &out[n++]))) return rc;
    }
  }
  *n_out = n;
  return KVT_OK;
}

typedef struct {
  int32_t ctx;
  int kind;
  cand_t target;
  double drop;
  int64_t bytes_freed;
} upd_t;

/* update_preferred proj/src/placement.cpp:165-170 */
static int upd_preferred(const upd_t* a, const upd_t* b) {
  if (a->drop != b->drop) return a->drop < b->drop;
  if (a->bytes_freed != b->bytes_freed) return a->bytes_freed > b->bytes_freed;
  if (a->ctx != b->ctx) return a->ctx < b->ctx;
  return 0;
}

/* least_drop_update proj/src/placement.cpp:174-204 */
static int least_drop(const kvt_store* s, int32_t ti, const kvt_pset* p, const space_t* sp,
                      double alpha, upd_t* best) {
  int rc, found = 0;
  cand_t opts[KVT_MAX_TIERS * (KVT_MAX_METHODS * KVT_MAX_RATIOS + 1)];
  const tierlist_t* L = &s->lists[ti];
  for (int32_t k = 0; k < L->n; ++k) {
    const int32_t c = L->ids[k];
    const kvt_entry* e = &s->e[c];
    cand_t cur;
    if ((rc = score(p, c, e->method, e->ratio, &s->tr, ti, sp, alpha, &cur))) return rc;
    int n;
    if ((rc = enumerate_updates(e, c, p, &s->tr, sp, alpha, opts, &n))) return rc;
    for (int j = 0; j < n; ++j) {
      upd_t u;
      u.ctx = c;
      u.kind = opts[j].tier_index == ti ? KVT_RECOMPRESS : KVT_EVICT;
      u.target = opts[j];
      u.drop = cur.utility - opts[j].utility;
      u.bytes_freed = u.kind == KVT_RECOMPRESS ? cur.size - opts[j].size : cur.size;
      if (!found || upd_preferred(&u, best)) {
        *best = u;
        found = 1;
      }
    }
  }
  if (!found)
    return orc_fail(KVT_EVALIDATION,
                    "tier %d is over capacity and no resident has a space-saving option",
                    s->tr.t[ti].tier_id);
  return KVT_OK;
}

int orc_least_drop_update(kvt_store* s, const kvt_pset* p, const kvt_space* space,
                          const kvt_params* params, int32_t tier_index, kvt_update* out) {
  space_t sp;
  int rc;
  if ((rc = resolve_space(space, &sp))) return rc;
  if (tier_index < 0 || tier_index >= s->tr.T) return orc_fail(KVT_EINVAL, "tier index");
  upd_t u;
  if ((rc = least_drop(s, tier_index, p, &sp, params->alpha, &u))) return rc;
  out->ctx = u.ctx;
  out->kind = u.kind;
  out->tier_index = u.target.tier_index;
  out->tier_id = u.target.tier_id;
  out->method = u.target.method;
  out->pad_ = 0;
  out->ratio = u.target.ratio;
  out->size_bytes = u.target.size;
  out->quality = u.target.quality;
  out->ttft = u.target.ttft;
  out->utility = u.target.utility;
  out->utility_drop = u.drop;
  out->bytes_freed = u.bytes_freed;
  return KVT_OK;
}

/* resolve_overflow proj/src/placement.cpp:206-223 */
static int resolve(kvt_store* s, const kvt_pset* p, const space_t* sp, double alpha) {
  int t, rc;
  while ((t = first_over(s)) >= 0) {
    upd_t u;
    if ((rc = least_drop(s, t, p, sp, alpha, &u))) return rc;
    if (u.kind == KVT_RECOMPRESS) {
      if ((rc = orc_store_reconfigure(s, u.ctx, u.target.method, u.target.ratio))) return rc;
    } else {
      kvt_entry moved;
      orc_store_remove(s, u.ctx, &moved);
      moved.tier_index = u.target.tier_index;
      moved.method = u.target.method;
      moved.ratio = u.target.ratio;
      if ((rc = orc_store_add(s, u.ctx, &moved))) return rc;
    }
    push_action(s, u.kind, u.ctx, u.target.tier_id, u.target.method, u.target.ratio);
  }
  return KVT_OK;
}

int orc_resolve_overflow(kvt_store* s, const kvt_pset* p, const kvt_space* space,
                         const kvt_params* params, int64_t* n_actions) {
  space_t sp;
  int rc;
  s->n_act = 0;
  if ((rc = resolve_space(space, &sp))) return rc;
  rc = resolve(s, p, &sp, params->alpha);
  *n_actions = s->n_act;
  return rc;
}

/* insert_joint proj/src/placement.cpp:225-250 */
static int insert_one(kvt_store* s, const kvt_pset* p, const space_t* sp, double alpha, int rule,
                      int32_t c, int64_t freq, int64_t stamp) {
  int rc;
  if ((rc = check_ctx(s, c))) return rc;
  if (s->e[c].tier_index >= 0) return orc_fail(KVT_EVALIDATION, "context %d is already resident", c);
  cand_t b;
  int32_t br;
  if ((rc = best_one(p, c, &s->tr, sp, alpha, rule, &b, &br))) return rc;
  kvt_entry e;
  memset(&e, 0, sizeof e);
  e.tier_index = b.tier_index;
  e.method = b.method;
  e.ratio = b.ratio;
  e.original_size_bytes = p->orig[c];
  e.frequency = freq;
  e.last_access = stamp;
  if ((rc = orc_store_add(s, c, &e))) return rc;
  push_action(s, KVT_INSERT, c, b.tier_id, b.method, b.ratio);
  return resolve(s, p, sp, alpha);
}

int orc_insert_joint(kvt_store* s, const kvt_pset* p, const kvt_space* space,
                     const kvt_params* params, int32_t rule, const int32_t* ctx,
                     const int64_t* frequency, const int64_t* stamp, int64_t n_ops,
                     int64_t* n_actions, int64_t* n_done) {
  space_t sp;
  int rc;
  s->n_act = 0;
  *n_done = 0;
  if ((rc = resolve_space(space, &sp))) {
    *n_actions = 0;
    return rc;
  }
  if (p->M != sp.M) return orc_fail(KVT_EINVAL, "method count mismatch");
  for (int64_t i = 0; i < n_ops; ++i) {
    rc = insert_one(s, p, &sp, params->alpha, rule, ctx[i], frequency ? frequency[i] : 0,
                    stamp ? stamp[i] : 0);
    if (rc) {
      *n_actions = s->n_act;
      return rc;
    }
    *n_done = i + 1;
  }
  *n_actions = s->n_act;
  return KVT_OK;
}

typedef struct {
  int32_t ctx;
  int64_t freq, stamp;
  double util;
} saved_t;

static int cmp_saved(const void* a, const void* b) {
  const saved_t* x = (const saved_t*)a;
  const saved_t* y = (const saved_t*)b;
  if (x->util != y->util) return x->util > y->util ? -1 : 1;
  return x->ctx < y->ctx ? -1 : (x->ctx > y->ctx ? 1 : 0);
}

/* rearrange proj/src/placement.cpp:252-283 (the comparator is a total order
 * on distinct contexts, so qsort gives the stable_sort result) */
int orc_rearrange(kvt_store* s, const kvt_pset* p, const kvt_space* space, const kvt_params* params,
                  int32_t rule, int64_t* n_actions) {
  space_t sp;
  int rc;
  s->n_act = 0;
  *n_actions = 0;
  if ((rc = resolve_space(space, &sp))) return rc;
  int32_t n = 0;
  for (int t = 0; t < s->tr.T; ++t) n += s->lists[t].n;
  saved_t* sv = (saved_t*)malloc(sizeof(saved_t) * (size_t)(n ? n : 1));
  int32_t k = 0;
  for (int t = 0; t < s->tr.T; ++t)
    for (int32_t i = 0; i < s->lists[t].n; ++i) {
      const int32_t c = s->lists[t].ids[i];
      cand_t b;
      int32_t br;
      if ((rc = best_one(p, c, &s->tr, &sp, params->alpha, rule, &b, &br))) {
        free(sv);
        return rc;
      }
      sv[k].ctx = c;
      sv[k].freq = s->e[c].frequency;
      sv[k].stamp = s->e[c].last_access;
      sv[k].util = b.utility;
      ++k;
    }
  qsort(sv, (size_t)n, sizeof(saved_t), cmp_saved);
  orc_store_clear(s);
  for (int32_t i = 0; i < n; ++i) {
    if ((rc = insert_one(s, p, &sp, params->alpha, rule, sv[i].ctx, sv[i].freq, sv[i].stamp))) {
      free(sv);
      *n_actions = s->n_act;
      return rc;
    }
  }
  free(sv);
  *n_actions = s->n_act;
  return KVT_OK;
}

/* placement_utility proj/src/placement.cpp:285-298 */
int orc_placement_utility(kvt_store* s, const kvt_pset* p, const kvt_space* space,
                          const kvt_params* params, double* out) {
  space_t sp;
  int rc;
  if ((rc = resolve_space(space, &sp))) return rc;
  double total = 0.0;
  for (int t = 0; t < s->tr.T; ++t)
    for (int32_t i = 0; i < s->lists[t].n; ++i) {
      const int32_t c = s->lists[t].ids[i];
      const kvt_entry* e = &s->e[c];
      double q;
      int64_t b;
      if ((rc = quality_of(p, c, e->method, &sp, e->ratio, &q))) return rc;
      if ((rc = csize(e->original_size_bytes, e->ratio, &b))) return rc;
      const double tt = load_time(b, &s->tr.t[t], sp.ovh[e->method]);
      total += utility_score(q, tt, p->freq[c], params->alpha);
    }
  *out = total;
  return KVT_OK;
}

int orc_store_bind_space(kvt_store* s, const kvt_space* space) {
  space_t sp;
  (void)s;
  return resolve_space(space, &sp);
}

/* tier moves, CPU restatement: every move is a plain memcpy of host memory
 * (test infrastructure: the same batch semantics as kvt_tier_moves) */
int orc_tier_moves(kvt_handle* h, const kvt_move* moves, int64_t n) {
  (void)h;
  for (int64_t i = 0; i < n; ++i) {
    if (moves[i].bytes < 0 || (moves[i].bytes > 0 && (!moves[i].src || !moves[i].dst))) return KVT_EINVAL;
    if (moves[i].bytes) memcpy(moves[i].dst, moves[i].src, (size_t)moves[i].bytes);
  }
  return KVT_OK;
}
