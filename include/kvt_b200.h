/*
 * kvt_b200.h — C ABI of the B200 EvicPress hot path.
 *
 * This is the drop-in boundary. The reference (`kvtier`, a C++20 library)
 * exposes its hot path as free functions in namespace kvtier
 * (proj/include/kvtier/utility.hpp, proj/include/kvtier/placement.hpp).
 * Every entry point below names the reference function it replaces.
 * Signatures use plain pointers, sizes and POD structs only: no torch,
 * no std:: types, no CUDA types. Three implementations share this ABI:
 *
 *   kvt_*   libkvt_b200.so      sm_100a CUDA (the product)
 *   orc_*   oracle/liboracle.so  CPU restatement (test infrastructure only)
 *   ref_*   oracle/_ref/libkvtier_ref.so  the reference library itself,
 *                                built from /root/reference sources
 *
 * Conventions
 *  - Contexts are identified by their index in byte-lexicographic order
 *    of ContextId (the iteration order of kvtier::ProfileMap, a
 *    std::map<std::string,...>). Tie-breaks "smaller context id" in the
 *    reference therefore become "smaller index".
 *  - Methods are identified by their index in the CandidateSpace's
 *    MethodSet insertion order (proj/src/utility.cpp:102,136).
 *  - Ratios are identified by their index in CandidateSpace order:
 *    sorted descending, de-duplicated (proj/src/utility.cpp:31-32).
 *  - Tiers are validated and stable-sorted by tier_id exactly like
 *    validate_hierarchy (proj/src/core.cpp:86-121); "tier index" is the
 *    position after sorting, actions report tier_id.
 *  - Every call returns a kvt_status; on failure kvt_last_error() (or
 *    orc_/ref_ equivalent) holds the message. KVT_EVALIDATION maps back to
 *    kvtier::ValidationError (proj/include/kvtier/core.hpp:18-20).
 *  - Functions are re-entrant per handle; one handle per thread/stream
 *    (the reference runs independent stores concurrently under
 *    `compare --jobs`, proj/tools/kvtier_main.cpp:206-235).
 */
#ifndef KVT_B200_H
#define KVT_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVT_ABI_VERSION 2

/* Hard limits of the device kernels (kernel-parameter structs). */
#define KVT_MAX_TIERS 8
#define KVT_MAX_METHODS 16
#define KVT_MAX_RATIOS 32

typedef enum {
  KVT_OK = 0,
  KVT_EVALIDATION = 1, /* kvtier::ValidationError */
  KVT_ETRACE = 2,      /* kvtier::TraceError */
  KVT_ECUDA = 3,       /* CUDA runtime / launch failure */
  KVT_EINVAL = 4,      /* bad ABI argument (null pointer, limits) */
  KVT_ENOMEM = 5
} kvt_status;

typedef enum { KVT_RULE_UTILITY = 0, KVT_RULE_QUALITY_FIRST = 1 } kvt_rule;
/* proj/include/kvtier/utility.hpp:87 SelectionRule */

typedef enum { KVT_INSERT = 0, KVT_RECOMPRESS = 1, KVT_EVICT = 2 } kvt_action_kind;
/* proj/include/kvtier/core.hpp:96-103 PlacementAction::Kind */

/* proj/include/kvtier/core.hpp:63-71 TierSpec (name dropped: only used in
 * error text). */
typedef struct {
  int32_t tier_id;
  int32_t unlimited; /* 1 = capacity_bytes is nullopt */
  int64_t capacity_bytes;
  double read_bandwidth;       /* bytes per second, > 0 */
  double fixed_access_latency; /* seconds, >= 0 */
} kvt_tier;

/* proj/include/kvtier/utility.hpp:31-46 CandidateSpace +
 * proj/include/kvtier/core.hpp:28-47 MethodSet. */
typedef struct {
  int32_t n_methods;
  const char* const* method_names;      /* insertion order */
  const double* decompression_overhead; /* seconds per byte, >= 0 */
  int32_t n_ratios;
  const double* ratios; /* any order; sorted desc + de-duplicated inside */
} kvt_space;

/* proj/include/kvtier/core.hpp:74-79 UtilityParams (prefill terms are not on
 * the placement path). */
typedef struct {
  double alpha;
} kvt_params;

/* A set of kvtier::ContextProfile (proj/include/kvtier/quality.hpp:20-29),
 * struct-of-arrays over contexts in ProfileMap order. Quality rows are
 * stored per *space* method (methods absent from the space are dropped,
 * they can never be enumerated; methods of the space absent from the
 * profile have has_method = 0 and are unscorable,
 * proj/src/utility.cpp:13-17). */
typedef struct {
  int32_t n_ctx;
  int32_t n_methods;                  /* == space n_methods */
  const int64_t* original_size_bytes; /* [n_ctx] */
  const double* frequency;            /* [n_ctx] profile frequency (utility.cpp:76) */
  const int32_t* grid_offset;         /* [n_ctx+1] CSR into grid */
  const double* grid;                 /* ascending ratio grid per context */
  const double* quality;  /* [grid_offset[c]*n_methods + m*len_c + i] */
  const uint8_t* has_method; /* [n_ctx*n_methods] */
} kvt_profiles;

/* proj/include/kvtier/core.hpp:96-103 PlacementAction. */
typedef struct {
  int32_t kind;    /* kvt_action_kind */
  int32_t ctx;     /* context index */
  int32_t tier_id; /* target tier id (current tier for Recompress) */
  int32_t method;  /* space method index */
  double ratio;
} kvt_action;

/* proj/include/kvtier/placement.hpp:75-81 UpdateCandidate with its
 * ConfigCandidate target (proj/include/kvtier/utility.hpp:17-26). */
typedef struct {
  int32_t ctx;
  int32_t kind; /* KVT_RECOMPRESS or KVT_EVICT */
  int32_t tier_index;
  int32_t tier_id;
  int32_t method;
  int32_t pad_;
  double ratio;
  int64_t size_bytes;
  double quality;
  double ttft;
  double utility;
  double utility_drop;
  int64_t bytes_freed;
} kvt_update;

/* Dense candidate tables (the all_candidates cross product,
 * proj/src/utility.cpp:129-145) laid out for the device:
 *   size    [n_ctx][R]          compressed_size(orig, ratio_r)
 *   quality [n_ctx][M][R]       quality_of; valid = scorable
 *   valid   [n_ctx][M][R]
 *   ttft    [n_ctx][T][M][R]    load_time
 *   utility [n_ctx][T][M][R]    utility_score
 * Any output pointer may be NULL. */

/* Per-context winner of best_config (proj/src/utility.cpp:159-172). */
typedef struct {
  int32_t status; /* 0 ok, 1 no scorable configuration (ValidationError) */
  int32_t tier_index;
  int32_t tier_id;
  int32_t method;
  int32_t ratio_index;
  int32_t pad_;
  double ratio;
  int64_t size_bytes;
  double quality;
  double ttft;
  double utility;
} kvt_best;

/* Resident snapshot of one context (proj/include/kvtier/core.hpp:84-93
 * CacheEntry). tier_index = -1 when not resident. seq orders arrival
 * within a tier (StoreState keeps per-tier vectors in arrival order). */
typedef struct {
  int32_t tier_index;
  int32_t method;
  double ratio;
  int64_t original_size_bytes;
  int64_t frequency;
  int64_t last_access;
  int64_t seq;
} kvt_entry;

typedef struct kvt_handle kvt_handle;   /* device, stream, scratch */
typedef struct kvt_pset kvt_pset;       /* uploaded profile set */
typedef struct kvt_store kvt_store;     /* StoreState */

#define KVT_DECLARE_API(P)                                                         \
  const char* P##last_error(void);                                                 \
  int P##abi_version(void);                                                        \
  /* handle: device ordinal, CUDA stream (NULL = default); CPU impls ignore */     \
  int P##create(int device, void* stream, kvt_handle** out);                       \
  int P##destroy(kvt_handle* h);                                                   \
  int P##pset_create(kvt_handle* h, const kvt_profiles* profiles, kvt_pset** out); \
  int P##pset_destroy(kvt_pset* p);                                                \
  /* utility.cpp:129-145 all_candidates (dense, all contexts) */                   \
  int P##score_candidates(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, \
                          int32_t n_tiers, const kvt_space* space,                 \
                          const kvt_params* params, int64_t* size, double* quality, \
                          uint8_t* valid, double* ttft, double* utility);          \
  /* utility.cpp:159-172 best_config (every context) */                            \
  int P##best_config(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers,      \
                     int32_t n_tiers, const kvt_space* space,                      \
                     const kvt_params* params, int32_t rule, kvt_best* out);       \
  /* placement.cpp:44-159 StoreState */                                            \
  int P##store_create(kvt_handle* h, const kvt_tier* tiers, int32_t n_tiers,       \
                      int32_t n_ctx, kvt_store** out);                             \
  int P##store_destroy(kvt_store* s);                                              \
  /* names entry method indices (store_add before any placement call) */          \
  int P##store_bind_space(kvt_store* s, const kvt_space* space);                   \
  int P##store_add(kvt_store* s, int32_t ctx, const kvt_entry* e);                 \
  int P##store_remove(kvt_store* s, int32_t ctx, kvt_entry* removed);              \
  int P##store_reconfigure(kvt_store* s, int32_t ctx, int32_t method, double ratio); \
  int P##store_touch(kvt_store* s, int32_t ctx, int64_t stamp);                    \
  /* n touches in order (the serve loop's hits; placement.cpp:135-142 each) */     \
  int P##store_touch_many(kvt_store* s, const int32_t* ctx, const int64_t* stamps, \
                          int64_t n);                                              \
  int P##store_clear(kvt_store* s);                                                \
  int P##store_occupancy(kvt_store* s, int64_t* occ);                              \
  int P##store_snapshot(kvt_store* s, kvt_entry* entries);                         \
  /* placement.cpp:174-204 least_drop_update (does not apply it) */                \
  int P##least_drop_update(kvt_store* s, const kvt_pset* p, const kvt_space* space, \
                           const kvt_params* params, int32_t tier_index,           \
                           kvt_update* out);                                       \
  /* placement.cpp:206-223 resolve_overflow. Actions of every mutating call   \
   * are buffered inside the store; *n_actions returns how many, fetch them  \
   * with store_actions. */                                                    \
  int P##resolve_overflow(kvt_store* s, const kvt_pset* p, const kvt_space* space, \
                          const kvt_params* params, int64_t* n_actions);           \
  /* placement.cpp:225-250 insert_joint, batched: ops applied in order, the    \
   * action list is the concatenation of the per-op lists. On error *n_done   \
   * tells how many ops completed (the failing op may be half applied, as in  \
   * the reference, which mutates before it throws). */                        \
  int P##insert_joint(kvt_store* s, const kvt_pset* p, const kvt_space* space,     \
                      const kvt_params* params, int32_t rule, const int32_t* ctx,  \
                      const int64_t* frequency, const int64_t* stamp, int64_t n_ops, \
                      int64_t* n_actions, int64_t* n_done);                        \
  /* placement.cpp:252-283 rearrange */                                            \
  int P##rearrange(kvt_store* s, const kvt_pset* p, const kvt_space* space,        \
                   const kvt_params* params, int32_t rule, int64_t* n_actions);    \
  /* copy the first n buffered actions of the last mutating call */               \
  int P##store_actions(kvt_store* s, kvt_action* out, int64_t n);                  \
  /* placement.cpp:285-298 placement_utility */                                    \
  int P##placement_utility(kvt_store* s, const kvt_pset* p, const kvt_space* space, \
                           const kvt_params* params, double* out);

KVT_DECLARE_API(kvt_)

/* ------------------------------------------------------------------------
 * KV codec (builder-defined; the reference has no codec, SPEC.md:15 —
 * parity unpinned). All pointers are device
 * pointers for kvt_*, host pointers for orc_*. Layout: K and V are bf16
 * [L][H][T][D] with D == 128.
 * ------------------------------------------------------------------------ */
typedef enum { KVT_SCORER_KNORM = 0, KVT_SCORER_KEYDIFF = 1, KVT_SCORER_SNAPKV = 2 } kvt_scorer;

typedef struct {
  int32_t L, H, T, D; /* D must be 128 */
} kvt_kv_shape;

/* kvt_codec_cfg.flags */
#define KVT_CODEC_KNORM_KEEP_LOW 1 /* knorm keeps LOW-norm keys (the cited knorm paper);
                                      default keeps high norms, dropping low */

/* One codec configuration resolved from a (method label, ratio) pair. */
typedef struct {
  int32_t scorer;     /* kvt_scorer */
  int32_t bits;       /* 2, 4, 8 or 16 (16 = bf16, token drop only) */
  int32_t keep;       /* tokens kept per (layer, kv head), 1..T */
  int32_t window;     /* snapkv observation window W (always kept) */
  int32_t q_heads;    /* snapkv query heads per kv head (GQA group) */
  int32_t pool;       /* snapkv max-pool kernel (odd) */
  int32_t flags;      /* KVT_CODEC_* bits */
  int32_t pad_;
  uint64_t q_seed;    /* snapkv synthetic query seed (used when no Q is passed) */
} kvt_codec_cfg;

/* Layout of one compressed chunk (all offsets in bytes from blob start). */
typedef struct {
  int64_t idx_off, idx_bytes;       /* int32 [L][H][keep] ascending */
  int64_t kcode_off, kcode_bytes;   /* u32 words, [L][H][keep][D*bits/32] */
  int64_t kscale_off, kzero_off, kparam_bytes; /* fp16 [L][H][ceil(keep/G)][D] each */
  int64_t vcode_off, vcode_bytes;   /* u32 words, [L][H][keep][D*bits/32] */
  int64_t vscale_off, vzero_off, vparam_bytes; /* fp16 [L][H][keep] each */
  int64_t total_bytes;
  /* 1 for the identity configuration (every token kept at 16 bits): the
   * compressed chunk IS the source KV, so the blob has no bytes, compress
   * launches nothing and tier moves copy the source K/V directly. */
  int64_t identity;
} kvt_blob_map;

#define KVT_QGROUP 128 /* K per-channel quant group (kept tokens) */

#define KVT_DECLARE_CODEC(P)                                                          \
  /* resolve "<scorer>[-q<bits>]" + retained-size ratio into a codec config */      \
  int P##codec_plan(const char* method, double ratio, const kvt_kv_shape* shape,     \
                    kvt_codec_cfg* out);                                             \
  int P##blob_layout(const kvt_kv_shape* shape, const kvt_codec_cfg* cfg,            \
                     kvt_blob_map* out);                                          \
  /* synthetic KV: counter hash of (seed, ctx, layer, head, token, dim) */          \
  int P##kv_generate(kvt_handle* h, const kvt_kv_shape* shape, uint64_t seed,        \
                     uint64_t ctx, uint16_t* k, uint16_t* v);                        \
  /* per-(layer, head, token) float scores; larger = more important. q: snapkv's  \
   * observation-window queries, bf16 [L][H*q_heads][window][D] (the last       \
   * `window` query positions of every query head); NULL = the     \
   * synthetic queries of cfg->q_seed. Ignored by knorm / keydiff. */            \
  int P##token_scores(kvt_handle* h, const kvt_kv_shape* shape,                      \
                      const kvt_codec_cfg* cfg, const uint16_t* k, const uint16_t* q, \
                      float* scores);                                                \
  /* per (layer, head): `keep` largest scores, ties -> lower index, ascending */    \
  int P##topk(kvt_handle* h, const kvt_kv_shape* shape, const kvt_codec_cfg* cfg,    \
              const float* scores, int32_t* idx);                                    \
  /* gather kept tokens, quantise, pack into blob */                                 \
  int P##pack(kvt_handle* h, const kvt_kv_shape* shape, const kvt_codec_cfg* cfg,    \
              const uint16_t* k, const uint16_t* v, const int32_t* idx, void* blob); \
  /* unpack + dequantise into bf16 [L][H][keep][D]; identity blobs have no bytes \
   * to unpack (KVT_EINVAL: the source KV is the decompressed KV) */              \
  int P##unpack(kvt_handle* h, const kvt_kv_shape* shape, const kvt_codec_cfg* cfg,  \
                const void* blob, uint16_t* k_out, uint16_t* v_out);                 \
  /* scores + topk + pack in one call (workspace: scores + idx, see below);       \
   * q as for token_scores */                                                      \
  int P##compress(kvt_handle* h, const kvt_kv_shape* shape, const kvt_codec_cfg* cfg, \
                  const uint16_t* k, const uint16_t* v, const uint16_t* q,           \
                  void* workspace, void* blob);                                      \
  int64_t P##compress_workspace_bytes(const kvt_kv_shape* shape, const kvt_codec_cfg* cfg);

KVT_DECLARE_CODEC(kvt_)

/* kvt_compress over slices (layer, head) [s0, s0 + ns) of the chunk only,
 * same workspace and blob: compressing a chunk as a sequence of slice groups
 * gives the blob kvt_compress gives. knorm / keydiff (and keep == T) only;
 * the scoring pass leaves K in L2 for the pack of the same group, so groups
 * of <= ~64 MB of K are read from HBM once. snapkv: KVT_EINVAL. */
int kvt_compress_slices(kvt_handle* h, const kvt_kv_shape* shape, const kvt_codec_cfg* cfg, const uint16_t* k,
                        const uint16_t* v, int32_t s0, int32_t ns, void* workspace, void* blob);

/* ------------------------------------------------------------------------
 * Tier-move executor: turns placement decisions
 * (PlacementAction, proj/include/kvtier/core.hpp:96-103; built at
 * proj/src/placement.cpp:213-221, only modelled by the reference)
 * into byte movement between the GPU tier (HBM) and the CPU tier (a pinned
 * host arena). A batch of moves is split into <= 8 MiB pieces spread over the
 * handle's copy streams (D2H and H2D use different copy engines, so the two
 * directions overlap); the batch starts after everything already queued on
 * the handle's stream (e.g. the compress that produced the blob) and the
 * handle's stream waits for its completion.
 * ------------------------------------------------------------------------ */
typedef enum { KVT_MOVE_D2H = 0, KVT_MOVE_H2D = 1, KVT_MOVE_D2D = 2, KVT_MOVE_H2H = 3 } kvt_move_kind;

typedef struct {
  const void* src;
  void* dst;
  int64_t bytes;
  int32_t kind; /* kvt_move_kind */
  int32_t pad_;
} kvt_move;

/* pinned (page-locked) host arena for the CPU tier */
int kvt_tier_host_alloc(int64_t bytes, void** out);
int kvt_tier_host_free(void* p);
int kvt_tier_moves(kvt_handle* h, const kvt_move* moves, int64_t n);
/* the CPU restatement: plain memcpy (host pointers only) */
int orc_tier_moves(kvt_handle* h, const kvt_move* moves, int64_t n);

/* SSD tier: pinned host pieces <-> a file (O_DIRECT when 4 KiB aligned, else
 * buffered), spread over `threads` worker threads; writes end with
 * fdatasync. The bytes reach the file through the CPU-tier staging arena
 * (HBM -> pinned DRAM by kvt_tier_moves, DRAM -> file here). */
typedef struct kvt_tier_file kvt_tier_file;
typedef struct {
  void* host;     /* pinned host memory */
  int64_t bytes;
  int64_t offset; /* file offset */
} kvt_file_io;
int kvt_tier_file_open(const char* path, int64_t bytes, kvt_tier_file** out); /* create, reserve */
int kvt_tier_file_direct(const kvt_tier_file* f); /* 1 if O_DIRECT is available on this file system */
int kvt_tier_file_close(kvt_tier_file* f);
int kvt_tier_file_write(kvt_tier_file* f, const kvt_file_io* ios, int64_t n, int32_t threads);
int kvt_tier_file_read(kvt_tier_file* f, const kvt_file_io* ios, int64_t n, int32_t threads);

/* ---- oracle_mckp (proj/src/placement.cpp:300-372): the exact
 * one-configuration-per-context optimum under the tier capacities, by
 * branch and bound over every context's candidates in candidate_preferred
 * order (the reference's DFS result: the maximal total utility, ties to
 * the lexicographically first assignment). The search runs on the GPU,
 * one subtree per thread. Fails (KVT_EVALIDATION) when the assignment space
 * exceeds max_assignments, a context has no scorable configuration, or no
 * assignment fits. out[n]: each context's chosen candidate. */
int kvt_oracle_mckp(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, int32_t n_tiers,
                    const kvt_space* space, const kvt_params* params, double max_assignments,
                    double* total_utility, kvt_best* out);
/* the reference's own oracle_mckp behind the same signature (test glue, oracle/_ref) */
int ref_oracle_mckp(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, int32_t n_tiers,
                    const kvt_space* space, const kvt_params* params, double max_assignments,
                    double* total_utility, kvt_best* out);

/* ---- Multi-GPU profile exchange. Contexts shard by rank; the
 * greedy's argmin spans every resident of a tier (proj/src/placement.cpp:
 * 179-197), so every rank needs every context's profile before placement.
 * Each rank packs its rows into one flat RECORD (host), the records are
 * all-gathered over NCCL (ncclAllGather / all_gather_into_tensor: equal
 * sizes, rank-major), and kvt_pset_merge builds the global profile set from
 * the gathered records ON THE DEVICE (concatenation in rank order + grid
 * offsets rebased by rank; no host round trip). Context index = rank *
 * n_ctx + local index, i.e. rank-major ids ("r000-...", "r001-...") in
 * byte-lexicographic ProfileMap order.
 *
 * Record layout (256-byte aligned sections, offsets from the record start):
 *   i64 original_size_bytes[n] | f64 frequency[n] | f64 grid[g] |
 *   f64 quality[g*M] | i32 grid_offset[n+1] (local, 0..g) | u8 has_method[n*M]
 * with n = n_ctx, g = grid_len = grid_offset[n], M = n_methods. */
int64_t kvt_pset_record_bytes(int32_t n_ctx, int32_t grid_len, int32_t n_methods);
/* host: validate `profiles` like pset_create and write its record */
int kvt_pset_record_pack(const kvt_profiles* profiles, void* record);
/* device: `records` = world records of equal (n_ctx, grid_len, n_methods),
 * rank-major (the all-gather output). *out: NULL to allocate a profile set,
 * or a set from an earlier merge of the same dimensions to refill in place
 * (stream-ordered, no allocation, no host synchronisation). */
int kvt_pset_merge(kvt_handle* h, const void* records, int32_t world, int32_t n_ctx, int32_t grid_len,
                   int32_t n_methods, kvt_pset** out);
/* the CPU restatement (host pointers) */
int64_t orc_pset_record_bytes(int32_t n_ctx, int32_t grid_len, int32_t n_methods);
int orc_pset_record_pack(const kvt_profiles* profiles, void* record);
int orc_pset_merge(kvt_handle* h, const void* records, int32_t world, int32_t n_ctx, int32_t grid_len,
                   int32_t n_methods, kvt_pset** out);

/* Device-pointer variants and timing helpers used by the bench. */
/* Synchronise the handle's stream. */
int kvt_sync(kvt_handle* h);
/* Set the stream used by subsequent launches on this handle. */
int kvt_set_stream(kvt_handle* h, void* stream);
/* Number of kernels this handle launched so far (evidence for gpu_launches). */
int64_t kvt_launch_count(kvt_handle* h);

#ifdef __cplusplus
}
#endif

#endif /* KVT_B200_H */
