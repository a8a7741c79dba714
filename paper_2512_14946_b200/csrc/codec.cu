// KV codec on sm_100a: synthetic KV, token scores (knorm / keydiff /
// snapkv), per-(layer, head) top-k, gather + quantise + pack, unpack +
// dequantise. Builder-defined spec; bit-exact to
// oracle/orc_codec.c for everything but snapkv's softmax (fp32 here,
// tolerance-checked).
//
// Memory-bound design: one bf16 row (128 channels = 256 B) is owned by a
// half-warp, one 16-byte vector load per lane; reductions over the row are
// in-register chunk sums + a 4-step half-warp butterfly, which is also the
// canonical FP64 reduction order of the spec (so no atomics, no order
// dependence). Grids are sized in multiples of the SM count.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <string>

#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>

#include "codec_common.cuh"
#include "kvt_common.cuh"

using namespace kvt;



static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (!g_num_sms) g_num_sms = 148;
  }
  return g_num_sms;
}

#define LAUNCHED(h)                      \
  do {                                   \
    (h)->launches++;                     \
    KVT_CUDA_TRY(cudaGetLastError());    \
  } while (0)

// ------------------------------------------------------------------ plan

extern "C" int kvt_codec_plan(const char* method, double ratio, const kvt_kv_shape* shape, kvt_codec_cfg* out) {
  if (!method || !shape || !out) return set_error(KVT_EINVAL, "null argument");
  if (!(ratio > 0.0) || ratio > 1.0) return set_error(KVT_EVALIDATION, "codec ratio must be in (0, 1]");
  if (shape->D != kD || shape->T <= 0 || shape->L <= 0 || shape->H <= 0)
    return set_error(KVT_EINVAL, "unsupported KV shape (D must be 128)");
  std::memset(out, 0, sizeof(*out));
  const char* dash = std::strstr(method, "-q");
  const size_t n = dash ? size_t(dash - method) : std::strlen(method);
  int bits = 16;
  if (dash) {
    bits = std::atoi(dash + 2);
    if (bits != 2 && bits != 4 && bits != 8)
      return set_error(KVT_EVALIDATION, std::string("unsupported bit width in ") + method);
  }
  const std::string sc(method, n);
  if (sc == "knorm") out->scorer = KVT_SCORER_KNORM;
  else if (sc == "keydiff") out->scorer = KVT_SCORER_KEYDIFF;
  else if (sc == "snapkv") out->scorer = KVT_SCORER_SNAPKV;
  else return set_error(KVT_EVALIDATION, std::string("unknown codec method ") + method);
  static const int widths[4] = {2, 4, 8, 16};
  int w = 0;
  while (widths[w] < bits) ++w;
  while (widths[w] < 16 && ratio > eff_bytes(widths[w])) ++w;
  out->bits = widths[w];
  const double keep = ratio / eff_bytes(out->bits);
  long long k = static_cast<long long>(std::floor(keep * double(shape->T) + 0.5));
  k = std::max(1LL, std::min<long long>(k, shape->T));
  out->window = shape->T < 32 ? shape->T : 32;
  out->q_heads = 4;
  out->pool = 7;
  out->q_seed = 0x5eed5eedull;
  if (out->scorer == KVT_SCORER_SNAPKV && k < out->window) k = out->window;
  out->keep = static_cast<int32_t>(k);
  return KVT_OK;
}

extern "C" int kvt_blob_layout(const kvt_kv_shape* s, const kvt_codec_cfg* c, kvt_blob_map* o) {
  blob_map(*s, *c, o);
  return KVT_OK;
}

static int64_t ws_scores(const kvt_kv_shape* s) { return al256(4LL * s->L * s->H * s->T); }
static int64_t ws_fixed(const kvt_kv_shape* s) { return al256(8LL * s->L * s->H * kD); }

extern "C" int64_t kvt_compress_workspace_bytes(const kvt_kv_shape* s, const kvt_codec_cfg* c) {
  return 2 * ws_scores(s) + ws_fixed(s) + al256(4LL * s->L * s->H * c->keep);
}

static int check_shape(const kvt_kv_shape* s, const kvt_codec_cfg* c) {
  if (!s || s->D != kD || s->L <= 0 || s->H <= 0 || s->T <= 0)
    return set_error(KVT_EINVAL, "unsupported KV shape (D must be 128)");
  if (c && (c->keep < 1 || c->keep > s->T)) return set_error(KVT_EINVAL, "keep out of range");
  if (c && c->bits != 2 && c->bits != 4 && c->bits != 8 && c->bits != 16)
    return set_error(KVT_EINVAL, "bits must be 2, 4, 8 or 16");
  return KVT_OK;
}

// ---------------------------------------------------------- synthetic KV

__global__ void __launch_bounds__(256) k_kv_generate(uint4* __restrict__ K, uint4* __restrict__ V, uint64_t n8,
                                                     uint64_t seed, uint64_t ctx) {
  const uint64_t n = n8 * 8;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n8; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t kw[4], vw[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t e0 = i * 8 + 2 * j, e1 = e0 + 1;
      const uint32_t k0 = synth_bf16(seed, ctx, e0, (e0 & 127) % 16 == 3);
      const uint32_t k1 = synth_bf16(seed, ctx, e1, (e1 & 127) % 16 == 3);
      const uint32_t v0 = synth_bf16(seed, ctx, n + e0, false);
      const uint32_t v1 = synth_bf16(seed, ctx, n + e1, false);
      kw[j] = k0 | (k1 << 16);
      vw[j] = v0 | (v1 << 16);
    }
    if (K) K[i] = make_uint4(kw[0], kw[1], kw[2], kw[3]);
    if (V) V[i] = make_uint4(vw[0], vw[1], vw[2], vw[3]);
  }
}

extern "C" int kvt_kv_generate(kvt_handle* h, const kvt_kv_shape* s, uint64_t seed, uint64_t ctx, uint16_t* k,
                               uint16_t* v) {
  int rc;
  if ((rc = check_shape(s, nullptr))) return rc;
  const uint64_t n8 = uint64_t(s->L) * s->H * s->T * s->D / 8;
  const int blocks = num_sms() * 8;
  k_kv_generate<<<blocks, 256, 0, h->stream>>>(reinterpret_cast<uint4*>(k), reinterpret_cast<uint4*>(v), n8, seed,
                                               ctx);
  LAUNCHED(h);
  return KVT_OK;
}

// --------------------------------------------------------------- scores

// Sum of squares of one lane's 8 channels (chunk of the canonical order).
__device__ __forceinline__ double chunk_sumsq(const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double a = double(bf2f(w[j] & 0xffffu)), b = double(bf2f(w[j] >> 16));
    acc = __dadd_rn(acc, __dmul_rn(a, a));
    acc = __dadd_rn(acc, __dmul_rn(b, b));
  }
  return acc;
}

// butterfly over the 16 chunk sums of a half-warp (strides 8, 4, 2, 1)
__device__ __forceinline__ double half_butterfly(double p) {
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) p = __dadd_rn(p, __shfl_xor_sync(0xffffffffu, p, off));
  return p;
}

constexpr int kUnroll = 4;

// knorm: squared L2 norm of every key (larger = keep).
__global__ void __launch_bounds__(256) k_knorm(const uint4* __restrict__ K, float* __restrict__ out, long long ntok) {
  const int l16 = threadIdx.x & 15;
  const long long hw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 4;
  const long long nhw = (gridDim.x * (long long)blockDim.x) >> 4;
  // loop bounds are warp-uniform (both half-warps run the same trip count)
  for (long long b0 = hw & ~1LL; b0 < ntok; b0 += nhw * kUnroll) {
    const long long t0 = b0 + (hw & 1);
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const long long t = t0 + u * nhw;
      v[u] = t < ntok ? __ldcs(K + t * 16 + l16) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const long long t = t0 + u * nhw;
      const double n2 = half_butterfly(chunk_sumsq(v[u]));
      if (t < ntok && l16 == 0) out[t] = __double2float_rn(n2);
    }
  }
}

constexpr double kFx = 1099511627776.0;  // 2^40 fixed-point scale
constexpr int kKdTokens = 256;           // tokens per block (16 half-warps x 16)

// keydiff pass 1: S[slice][d] = sum_t rint(x_td / |x_t| * 2^40) (exact int64)
__global__ void __launch_bounds__(256) k_keydiff_sum(const uint4* __restrict__ K, unsigned long long* __restrict__ S,
                                                     int T) {
  __shared__ long long part[16][kD];
  const int l16 = threadIdx.x & 15, hw = threadIdx.x >> 4;
  const int slice = blockIdx.y;
  const int t_begin = blockIdx.x * kKdTokens;
  const uint4* Ks = K + static_cast<size_t>(slice) * T * 16;
  long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int t_end = min(T, t_begin + kKdTokens);
  for (int b = t_begin + (hw & ~1); b < t_end; b += 16) {  // warp-uniform trip count
    const int t = b + (hw & 1);
    const uint4 v = t < t_end ? Ks[static_cast<size_t>(t) * 16 + l16] : make_uint4(0, 0, 0, 0);
    const double n2 = half_butterfly(chunk_sumsq(v));
    const double inv = n2 > 0.0 ? __drcp_rn(__dsqrt_rn(n2)) : 0.0;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double a = __dmul_rn(double(bf2f(w[j] & 0xffffu)), inv);
      const double b = __dmul_rn(double(bf2f(w[j] >> 16)), inv);
      acc[2 * j] += __double2ll_rn(__dmul_rn(a, kFx));
      acc[2 * j + 1] += __double2ll_rn(__dmul_rn(b, kFx));
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) part[hw][l16 * 8 + i] = acc[i];
  __syncthreads();
  if (threadIdx.x < kD) {
    long long s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += part[i][threadIdx.x];
    atomicAdd(S + static_cast<size_t>(slice) * kD + threadIdx.x, static_cast<unsigned long long>(s));
  }
}

// keydiff pass 2: score_t = -(khat_t . S) in the canonical FP64 order.
__global__ void __launch_bounds__(256) k_keydiff_score(const uint4* __restrict__ K,
                                                       const long long* __restrict__ S, float* __restrict__ out,
                                                       int T) {
  const int l16 = threadIdx.x & 15, hw = threadIdx.x >> 4;
  const int slice = blockIdx.y;
  const int t_begin = blockIdx.x * kKdTokens;
  const uint4* Ks = K + static_cast<size_t>(slice) * T * 16;
  double sd[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    sd[i] = __dmul_rn(__ll2double_rn(S[static_cast<size_t>(slice) * kD + l16 * 8 + i]), 1.0 / kFx);
  const int t_end = min(T, t_begin + kKdTokens);
  for (int b = t_begin + (hw & ~1); b < t_end; b += 16) {  // warp-uniform trip count
    const int t = b + (hw & 1);
    const uint4 v = t < t_end ? __ldcs(Ks + static_cast<size_t>(t) * 16 + l16) : make_uint4(0, 0, 0, 0);
    const double n2 = half_butterfly(chunk_sumsq(v));
    const double inv = n2 > 0.0 ? __drcp_rn(__dsqrt_rn(n2)) : 0.0;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double a = __dmul_rn(double(bf2f(w[j] & 0xffffu)), inv);
      const double b = __dmul_rn(double(bf2f(w[j] >> 16)), inv);
      acc = __dadd_rn(acc, __dmul_rn(a, sd[2 * j]));
      acc = __dadd_rn(acc, __dmul_rn(b, sd[2 * j + 1]));
    }
    const double p = half_butterfly(acc);
    if (l16 == 0 && t < t_end) out[static_cast<size_t>(slice) * T + t] = __double2float_rn(-p);
  }
}

// snapkv: observation window of W synthetic queries per
// q-head (GQA group G), softmax over the prefix, summed over the window and
// the group, then max-pooled; window tokens always kept (+inf).
// CUDA-core reference kernel: one block per (layer, kv head), one thread
// per query row, two passes (row stats, then probabilities).
constexpr int kSnapTile = 32;
__global__ void __launch_bounds__(128) k_snapkv_votes(const uint16_t* __restrict__ K, float* __restrict__ vote,
                                                      int L, int H, int T, int W, int G, uint64_t q_seed) {
  extern __shared__ float sm[];
  const int rows = W * G;
  float* q = sm;                                 // [rows][kD+1]
  float* kt = q + 128 * (kD + 1);                // [kSnapTile][kD]
  float* red = kt + kSnapTile * kD;              // [4][kSnapTile]
  const int slice = blockIdx.x, l = slice / H, h = slice % H;
  const int r = threadIdx.x, lane = r & 31, warp = r >> 5;
  const int P = T - W;
  const uint64_t Hq = uint64_t(H) * G;
  for (int i = threadIdx.x; i < rows * kD; i += blockDim.x) {
    const int rr = i / kD, d = i % kD, g = rr / W, w = rr % W;
    const uint64_t idx = ((uint64_t(l) * Hq + uint64_t(h * G + g)) * uint64_t(W) + uint64_t(w)) * kD + d;
    q[rr * (kD + 1) + d] = bf2f(synth_bf16(q_seed, 0x51ull, idx, d % 16 == 3));
  }
  const uint16_t* Ks = K + static_cast<size_t>(slice) * T * kD;
  const float scale = 1.0f / sqrtf(float(kD));
  float m = -INFINITY, lsum = 0.0f;
  for (int pass = 0; pass < 2; ++pass) {
    for (int t0 = 0; t0 < P; t0 += kSnapTile) {
      __syncthreads();
      for (int i = threadIdx.x; i < kSnapTile * kD; i += blockDim.x) {
        const int tt = t0 + i / kD;
        kt[i] = tt < P ? bf2f(Ks[static_cast<size_t>(tt) * kD + (i % kD)]) : 0.0f;
      }
      __syncthreads();
      const int nt = min(kSnapTile, P - t0);
      for (int j = 0; j < nt; ++j) {
        float s = 0.0f;
        if (r < rows) {
#pragma unroll 8
          for (int d = 0; d < kD; ++d) s = fmaf(q[r * (kD + 1) + d], kt[j * kD + d], s);
          s *= scale;
        }
        if (pass == 0) {
          if (r < rows) {
            if (s > m) {
              lsum = lsum * expf(m - s) + 1.0f;
              m = s;
            } else {
              lsum += expf(s - m);
            }
          }
        } else {
          float p = r < rows ? expf(s - m) / lsum : 0.0f;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
          if (lane == 0) red[warp * kSnapTile + j] = p;
        }
      }
      if (pass == 1) {
        __syncthreads();
        if (threadIdx.x < nt) {
          const float v = red[threadIdx.x] + red[kSnapTile + threadIdx.x] + red[2 * kSnapTile + threadIdx.x] +
                          red[3 * kSnapTile + threadIdx.x];
          vote[static_cast<size_t>(slice) * T + t0 + threadIdx.x] = v;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_snapkv_pool(const float* __restrict__ vote, float* __restrict__ out, int T,
                                                     int W, int pool) {
  const int slice = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int P = T - W, half = pool / 2;
  const float* v = vote + static_cast<size_t>(slice) * T;
  float r;
  if (t >= P) {
    r = INFINITY;
  } else {
    r = v[t];
    for (int j = max(0, t - half); j <= min(P - 1, t + half); ++j) r = fmaxf(r, v[j]);
  }
  out[static_cast<size_t>(slice) * T + t] = r;
}

static int launch_scores(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k,
                         float* scores, float* votes, unsigned long long* fixed) {
  const int S = s->L * s->H, T = s->T;
  cudaStream_t st = h->stream;
  if (c->scorer == KVT_SCORER_KNORM) {
    const long long ntok = static_cast<long long>(S) * T;
    const long long want = (ntok * 16 + 255) / 256;
    const int blocks = static_cast<int>(std::min<long long>(want, num_sms() * 16LL));
    k_knorm<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(k), scores, ntok);
    LAUNCHED(h);
  } else if (c->scorer == KVT_SCORER_KEYDIFF) {
    KVT_CUDA_TRY(cudaMemsetAsync(fixed, 0, 8LL * S * kD, st));
    dim3 grid((T + kKdTokens - 1) / kKdTokens, S);
    k_keydiff_sum<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(k), fixed, T);
    LAUNCHED(h);
    k_keydiff_score<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(k),
                                          reinterpret_cast<const long long*>(fixed), scores, T);
    LAUNCHED(h);
  } else if (c->scorer == KVT_SCORER_SNAPKV) {
    if (c->window * c->q_heads > 128 || c->window > T) return set_error(KVT_EINVAL, "snapkv window too large");
    const size_t smem = sizeof(float) * (128 * (kD + 1) + kSnapTile * kD + 4 * kSnapTile);
    static bool attr = false;
    if (!attr) {
      KVT_CUDA_TRY(cudaFuncSetAttribute(k_snapkv_votes, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr = true;
    }
    k_snapkv_votes<<<S, 128, smem, st>>>(k, votes, s->L, s->H, T, c->window, c->q_heads, c->q_seed);
    LAUNCHED(h);
    dim3 grid((T + 255) / 256, S);
    k_snapkv_pool<<<grid, 256, 0, st>>>(votes, scores, T, c->window, c->pool);
    LAUNCHED(h);
  } else {
    return set_error(KVT_EINVAL, "unknown scorer");
  }
  return KVT_OK;
}

static int ensure_scratch(kvt_handle* h, size_t bytes) {
  if (h->scratch_bytes >= bytes) return KVT_OK;
  if (h->scratch) cudaFree(h->scratch);
  h->scratch = nullptr;
  h->scratch_bytes = 0;
  KVT_CUDA_TRY(cudaMalloc(&h->scratch, bytes));
  h->scratch_bytes = bytes;
  return KVT_OK;
}

extern "C" int kvt_token_scores(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k,
                                float* scores) {
  int rc;
  if ((rc = check_shape(s, c))) return rc;
  if ((rc = ensure_scratch(h, ws_scores(s) + ws_fixed(s)))) return rc;
  char* b = static_cast<char*>(h->scratch);
  return launch_scores(h, s, c, k, scores, reinterpret_cast<float*>(b),
                       reinterpret_cast<unsigned long long*>(b + ws_scores(s)));
}

// ------------------------------------------------------------------ top-k

constexpr int kTopkThreads = 512;
using TopkScan = cub::BlockScan<int, kTopkThreads>;

// Per (layer, head): the `keep` largest scores, ties -> lower index,
// indices ascending. MSB-first 8-bit radix select on orderable keys held in
// shared memory, then an order-preserving block compaction.
__global__ void __launch_bounds__(kTopkThreads) k_topk(const float* __restrict__ scores, int32_t* __restrict__ idx,
                                                       int T, int k, int keys_in_smem) {
  extern __shared__ uint32_t skeys[];
  __shared__ int hist[256];
  __shared__ uint32_t s_prefix, s_mask;
  __shared__ int s_remaining;
  __shared__ typename TopkScan::TempStorage scan_tmp;
  const int slice = blockIdx.x, tid = threadIdx.x;
  const float* sc = scores + static_cast<size_t>(slice) * T;
  if (keys_in_smem)
    for (int t = tid; t < T; t += kTopkThreads) skeys[t] = score_key(sc[t]);
  if (tid == 0) {
    s_prefix = 0;
    s_mask = 0;
    s_remaining = k;
  }
  __syncthreads();
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += kTopkThreads) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix, mask = s_mask;
    for (int t = tid; t < T; t += kTopkThreads) {
      const uint32_t key = keys_in_smem ? skeys[t] : score_key(sc[t]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int rem = s_remaining, b = 255;
      for (; b > 0; --b) {
        if (hist[b] >= rem) break;
        rem -= hist[b];
      }
      s_remaining = rem;
      s_prefix = prefix | (uint32_t(b) << shift);
      s_mask = mask | (255u << shift);
    }
    __syncthreads();
  }
  const uint32_t kth = s_prefix;
  const int ties = s_remaining;  // equal-to-kth keys to take (lowest indices)
  const int seg = (T + kTopkThreads - 1) / kTopkThreads;
  const int t0 = tid * seg, t1 = min(T, t0 + seg);
  int above = 0, eq = 0;
  for (int t = t0; t < t1; ++t) {
    const uint32_t key = keys_in_smem ? skeys[t] : score_key(sc[t]);
    above += key > kth;
    eq += key == kth;
  }
  int above_before, eq_before;
  TopkScan(scan_tmp).ExclusiveSum(above, above_before);
  __syncthreads();
  TopkScan(scan_tmp).ExclusiveSum(eq, eq_before);
  int pos = above_before + min(eq_before, ties);
  int eq_seen = eq_before;
  int32_t* out = idx + static_cast<size_t>(slice) * k;
  for (int t = t0; t < t1; ++t) {
    const uint32_t key = keys_in_smem ? skeys[t] : score_key(sc[t]);
    if (key > kth) {
      out[pos++] = t;
    } else if (key == kth) {
      if (eq_seen < ties) out[pos++] = t;
      ++eq_seen;
    }
  }
}

static int launch_topk(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const float* scores,
                       int32_t* idx) {
  const int S = s->L * s->H;
  const size_t smem = sizeof(uint32_t) * size_t(s->T);
  const int in_smem = smem <= 160 * 1024;
  static bool attr = false;
  if (!attr) {
    KVT_CUDA_TRY(cudaFuncSetAttribute(k_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr = true;
  }
  k_topk<<<S, kTopkThreads, in_smem ? smem : 0, h->stream>>>(scores, idx, s->T, c->keep, in_smem);
  LAUNCHED(h);
  return KVT_OK;
}

extern "C" int kvt_topk(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const float* scores,
                        int32_t* idx) {
  int rc;
  if ((rc = check_shape(s, c))) return rc;
  return launch_topk(h, s, c, scores, idx);
}

// -------------------------------------------------------------------- pack

// bits == 16: gather kept K/V rows (half-warp per row, 16-byte lanes).
__global__ void __launch_bounds__(256) k_gather16(const uint4* __restrict__ K, const uint4* __restrict__ V,
                                                  const int32_t* __restrict__ idx, int32_t* __restrict__ oidx,
                                                  uint4* __restrict__ ko, uint4* __restrict__ vo, int T, int k) {
  const int slice = blockIdx.y, l16 = threadIdx.x & 15;
  const int j = blockIdx.x * 16 + (threadIdx.x >> 4);
  if (j >= k) return;
  const int t = idx[static_cast<size_t>(slice) * k + j];
  const size_t src = (static_cast<size_t>(slice) * T + t) * 16 + l16;
  const size_t dst = (static_cast<size_t>(slice) * k + j) * 16 + l16;
  const uint4 a = __ldcs(K + src), b = __ldcs(V + src);
  __stcs(ko + dst, a);
  __stcs(vo + dst, b);
  if (l16 == 0) oidx[static_cast<size_t>(slice) * k + j] = t;
}

// K quantisation: per channel over a group of <=128 kept tokens. The whole
// block (256 threads) packs group g of one slice: rows staged in smem,
// channel min/max split over two thread halves, codes packed row-wise with
// coalesced stores. Block-uniform: call from every thread.
struct PackKSmem {
  uint4 rows[KVT_QGROUP][16];        // 32 KB bf16 tile
  uint8_t codes[KVT_QGROUP][kD + 4];
  float pmn[2][kD], pmx[2][kD];
  QParam prm[kD];
};

__device__ __forceinline__ void pack_k_group(const uint4* __restrict__ K, const int32_t* __restrict__ idx,
                                             uint32_t* __restrict__ kc, uint16_t* __restrict__ ks,
                                             uint16_t* __restrict__ kz, int T, int k, int bits, int slice, int g,
                                             PackKSmem& sm) {
  const int tid = threadIdx.x;
  const int j0 = g * KVT_QGROUP, nr = min(KVT_QGROUP, k - j0);
  const int ng = (k + KVT_QGROUP - 1) / KVT_QGROUP;
  const int32_t* ix = idx + static_cast<size_t>(slice) * k + j0;
  for (int i = tid; i < nr * 16; i += 256) {
    const int r = i >> 4, l16 = i & 15;
    sm.rows[r][l16] = __ldcs(K + (static_cast<size_t>(slice) * T + ix[r]) * 16 + l16);
  }
  __syncthreads();
  const int d = tid & (kD - 1), half = tid >> 7;
  const uint16_t* tile = reinterpret_cast<const uint16_t*>(sm.rows);
  {
    const int r0 = half * 64, r1 = min(nr, r0 + 64);
    float mn = INFINITY, mx = -INFINITY;
    for (int r = r0; r < r1; ++r) {
      const float x = bf2f(tile[r * kD + d]);
      mn = x < mn ? x : mn;
      mx = x > mx ? x : mx;
    }
    sm.pmn[half][d] = mn;
    sm.pmx[half][d] = mx;
  }
  __syncthreads();
  if (half == 0) {
    const float mn = sm.pmn[1][d] < sm.pmn[0][d] ? sm.pmn[1][d] : sm.pmn[0][d];
    const float mx = sm.pmx[1][d] > sm.pmx[0][d] ? sm.pmx[1][d] : sm.pmx[0][d];
    const QParam p = make_param(mn, mx, bits);
    sm.prm[d] = p;
    const size_t po = (static_cast<size_t>(slice) * ng + g) * kD + d;
    ks[po] = p.s16;
    kz[po] = p.z16;
  }
  __syncthreads();
  {
    const QParam p = sm.prm[d];
    const int r0 = half * 64, r1 = min(nr, r0 + 64);
    for (int r = r0; r < r1; ++r) sm.codes[r][d] = static_cast<uint8_t>(quant(bf2f(tile[r * kD + d]), p, bits));
  }
  __syncthreads();
  const int wpr = kD * bits / 32, per = 32 / bits;
  uint32_t* out = kc + (static_cast<size_t>(slice) * k + j0) * wpr;
  for (int i = tid; i < nr * wpr; i += 256) {
    const int r = i / wpr, w = i - r * wpr;
    uint32_t word = 0;
    for (int q = 0; q < per; ++q) word |= uint32_t(sm.codes[r][w * per + q]) << (bits * q);
    out[i] = word;
  }
  __syncthreads();  // smem reused by the next group
}

__global__ void __launch_bounds__(256) k_pack_k(const uint4* __restrict__ K, const int32_t* __restrict__ idx,
                                                uint32_t* __restrict__ kc, uint16_t* __restrict__ ks,
                                                uint16_t* __restrict__ kz, int T, int k, int bits) {
  extern __shared__ uint4 pack_smem[];
  pack_k_group(K, idx, kc, ks, kz, T, k, bits, blockIdx.y, blockIdx.x, *reinterpret_cast<PackKSmem*>(pack_smem));
}

// V quantisation: per kept token over its 128 channels; half-warp per row.
// Warp-uniform: both half-warps must call (shuffles use the full mask).
__device__ __forceinline__ void pack_v_row(const uint4* __restrict__ V, const int32_t* __restrict__ idx,
                                           int32_t* __restrict__ oidx, uint32_t* __restrict__ vc,
                                           uint16_t* __restrict__ vs, uint16_t* __restrict__ vz, int T, int k,
                                           int bits, int slice, int j) {
  const int l16 = threadIdx.x & 15;
  const bool live = j < k;
  const int t = live ? idx[static_cast<size_t>(slice) * k + j] : 0;
  const uint4 v = live ? __ldcs(V + (static_cast<size_t>(slice) * T + t) * 16 + l16) : make_uint4(0, 0, 0, 0);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  float x[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[2 * i] = bf2f(w[i] & 0xffffu);
    x[2 * i + 1] = bf2f(w[i] >> 16);
  }
  float mn = x[0], mx = x[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    mn = x[i] < mn ? x[i] : mn;
    mx = x[i] > mx ? x[i] : mx;
  }
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) {
    const float a = __shfl_xor_sync(0xffffffffu, mn, off), b = __shfl_xor_sync(0xffffffffu, mx, off);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  const QParam p = make_param(mn, mx, bits);
  uint32_t c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = quant(x[i], p, bits);
  const int wpr = kD * bits / 32;
  uint32_t* out = vc + (static_cast<size_t>(slice) * k + j) * wpr;
  if (bits == 8) {
    const uint32_t w0 = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
    const uint32_t w1 = c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24);
    if (live) __stcs(reinterpret_cast<uint2*>(out) + l16, make_uint2(w0, w1));
  } else if (bits == 4) {
    uint32_t w0 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w0 |= c[i] << (4 * i);
    if (live) __stcs(out + l16, w0);
  } else {  // 2 bits: 16 codes per word = two lanes
    uint32_t h0 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) h0 |= c[i] << (2 * i);
    const uint32_t other = __shfl_xor_sync(0xffffffffu, h0, 1);
    if (live && (l16 & 1) == 0) __stcs(out + (l16 >> 1), h0 | (other << 16));
  }
  if (live && l16 == 0) {
    vs[static_cast<size_t>(slice) * k + j] = p.s16;
    vz[static_cast<size_t>(slice) * k + j] = p.z16;
    if (oidx) oidx[static_cast<size_t>(slice) * k + j] = t;
  }
}

__global__ void __launch_bounds__(256) k_pack_v(const uint4* __restrict__ V, const int32_t* __restrict__ idx,
                                                int32_t* __restrict__ oidx, uint32_t* __restrict__ vc,
                                                uint16_t* __restrict__ vs, uint16_t* __restrict__ vz, int T, int k,
                                                int bits) {
  pack_v_row(V, idx, oidx, vc, vs, vz, T, k, bits, blockIdx.y, blockIdx.x * 16 + (threadIdx.x >> 4));
}

static int launch_pack(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k,
                       const uint16_t* v, const int32_t* idx, void* blob) {
  kvt_blob_map m;
  blob_map(*s, *c, &m);
  char* b = static_cast<char*>(blob);
  const int S = s->L * s->H, kk = c->keep;
  cudaStream_t st = h->stream;
  dim3 rows_grid((kk + 15) / 16, S);
  if (c->bits == 16) {
    k_gather16<<<rows_grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(k), reinterpret_cast<const uint4*>(v), idx,
                                          reinterpret_cast<int32_t*>(b + m.idx_off),
                                          reinterpret_cast<uint4*>(b + m.kcode_off),
                                          reinterpret_cast<uint4*>(b + m.vcode_off), s->T, kk);
    LAUNCHED(h);
    return KVT_OK;
  }
  dim3 kgrid((kk + KVT_QGROUP - 1) / KVT_QGROUP, S);
  const size_t pk_smem = sizeof(PackKSmem);
  static bool pk_attr = false;
  if (!pk_attr) {
    KVT_CUDA_TRY(cudaFuncSetAttribute(k_pack_k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pk_smem)));
    pk_attr = true;
  }
  k_pack_k<<<kgrid, 256, pk_smem, st>>>(reinterpret_cast<const uint4*>(k), idx, reinterpret_cast<uint32_t*>(b + m.kcode_off),
                                  reinterpret_cast<uint16_t*>(b + m.kscale_off),
                                  reinterpret_cast<uint16_t*>(b + m.kzero_off), s->T, kk, c->bits);
  LAUNCHED(h);
  k_pack_v<<<rows_grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(v), idx, reinterpret_cast<int32_t*>(b + m.idx_off),
                                      reinterpret_cast<uint32_t*>(b + m.vcode_off),
                                      reinterpret_cast<uint16_t*>(b + m.vscale_off),
                                      reinterpret_cast<uint16_t*>(b + m.vzero_off), s->T, kk, c->bits);
  LAUNCHED(h);
  return KVT_OK;
}

extern "C" int kvt_pack(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k,
                        const uint16_t* v, const int32_t* idx, void* blob) {
  int rc;
  if ((rc = check_shape(s, c))) return rc;
  return launch_pack(h, s, c, k, v, idx, blob);
}

// ------------------------------------------------------------------ unpack

__global__ void __launch_bounds__(256) k_unpack(const uint8_t* __restrict__ blob, kvt_blob_map m,
                                                uint4* __restrict__ ko, uint4* __restrict__ vo, int k, int bits) {
  const int slice = blockIdx.y, l16 = threadIdx.x & 15;
  const int j = blockIdx.x * 16 + (threadIdx.x >> 4);
  if (j >= k) return;
  const size_t row = static_cast<size_t>(slice) * k + j;
  const int wpr = kD * bits / 32, ng = (k + KVT_QGROUP - 1) / KVT_QGROUP, g = j / KVT_QGROUP;
  const uint32_t* kc = reinterpret_cast<const uint32_t*>(blob + m.kcode_off) + row * wpr;
  const uint32_t* vc = reinterpret_cast<const uint32_t*>(blob + m.vcode_off) + row * wpr;
  const uint16_t* ks = reinterpret_cast<const uint16_t*>(blob + m.kscale_off) + (static_cast<size_t>(slice) * ng + g) * kD;
  const uint16_t* kz = reinterpret_cast<const uint16_t*>(blob + m.kzero_off) + (static_cast<size_t>(slice) * ng + g) * kD;
  const float vsf = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(blob + m.vscale_off)[row]));
  const float vzf = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(blob + m.vzero_off)[row]));
  const uint32_t mask = (1u << bits) - 1u;
  const int per = 32 / bits;
  uint32_t ok[4], ov[4];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    uint32_t pk[2], pv[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int d = l16 * 8 + i + e;
      const uint32_t kcode = (kc[d / per] >> (bits * (d % per))) & mask;
      const uint32_t vcode = (vc[d / per] >> (bits * (d % per))) & mask;
      pk[e] = dequant_bf16(kcode, __half2float(__ushort_as_half(ks[d])), __half2float(__ushort_as_half(kz[d])));
      pv[e] = dequant_bf16(vcode, vsf, vzf);
    }
    ok[i / 2] = pk[0] | (pk[1] << 16);
    ov[i / 2] = pv[0] | (pv[1] << 16);
  }
  ko[row * 16 + l16] = make_uint4(ok[0], ok[1], ok[2], ok[3]);
  vo[row * 16 + l16] = make_uint4(ov[0], ov[1], ov[2], ov[3]);
}

extern "C" int kvt_unpack(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const void* blob,
                          uint16_t* k_out, uint16_t* v_out) {
  int rc;
  if ((rc = check_shape(s, c))) return rc;
  kvt_blob_map m;
  blob_map(*s, *c, &m);
  const int S = s->L * s->H, kk = c->keep;
  const char* b = static_cast<const char*>(blob);
  if (c->bits == 16) {
    KVT_CUDA_TRY(cudaMemcpyAsync(k_out, b + m.kcode_off, m.kcode_bytes, cudaMemcpyDeviceToDevice, h->stream));
    KVT_CUDA_TRY(cudaMemcpyAsync(v_out, b + m.vcode_off, m.vcode_bytes, cudaMemcpyDeviceToDevice, h->stream));
    return KVT_OK;
  }
  dim3 grid((kk + 15) / 16, S);
  k_unpack<<<grid, 256, 0, h->stream>>>(reinterpret_cast<const uint8_t*>(blob), m, reinterpret_cast<uint4*>(k_out),
                                        reinterpret_cast<uint4*>(v_out), kk, c->bits);
  LAUNCHED(h);
  return KVT_OK;
}


// ------------------------------------------------------- fused compress
//
// One thread-block cluster of kFuseC CTAs per (layer, kv-head) slice does
// scores -> top-k -> gather + quantise + pack in a single launch. Each CTA
// owns a contiguous token range of the slice. Cross-CTA steps go through
// distributed shared memory: keydiff's mean direction (exact int64 fixed
// point, so the sum order does not matter), the four radix-select
// histograms and the (above, equal) counts that place each CTA's kept
// indices. Only kFuseC x (#clusters in flight) slices are live at a time
// (~40 x 2 MiB of K at T = 8192), so the re-reads of K (keydiff's second
// pass, the kept rows in the pack) are L2 hits: HBM sees K once, the kept V
// rows once and the blob once. Bit-identical to the unfused kernels.
namespace cg = cooperative_groups;
constexpr int kFuseC = 8;
constexpr int kFuseThreads = 256;
constexpr int kFuseUnroll = 4;
constexpr size_t kFuseUnion = sizeof(PackKSmem) > 16 * kD * sizeof(long long) ? sizeof(PackKSmem)
                                                                                : 16 * kD * sizeof(long long);
constexpr size_t kFuseMaxSmem = 200 * 1024;
using FuseScan = cub::BlockScan<int, kFuseThreads>;

static size_t fuse_smem_bytes(int T) {
  const size_t per = (T + kFuseC - 1) / kFuseC;
  return kFuseUnion + al256(4 * per);
}

__global__ void __cluster_dims__(kFuseC, 1, 1) __launch_bounds__(kFuseThreads, 2)
    k_compress_fused(const uint4* __restrict__ K, const uint4* __restrict__ V, int T, int k, int bits, int scorer,
                     kvt_blob_map m, char* __restrict__ blob) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  const int slice = blockIdx.y, tid = threadIdx.x, l16 = tid & 15, hw = tid >> 4;
  const int per = (T + kFuseC - 1) / kFuseC;
  const int t_lo = min(T, rank * per), t_hi = min(T, t_lo + per), n_loc = t_hi - t_lo;
  extern __shared__ __align__(16) uint8_t fsm[];
  PackKSmem& pk = *reinterpret_cast<PackKSmem*>(fsm);
  long long(*part)[kD] = reinterpret_cast<long long(*)[kD]>(fsm);
  uint32_t* keys = reinterpret_cast<uint32_t*>(fsm + kFuseUnion);
  __shared__ int hist[2][256];
  __shared__ int tot[256];
  __shared__ long long sfix[kD];
  __shared__ double sdir[kD];
  __shared__ int cnt[2];
  __shared__ uint32_t s_prefix, s_mask;
  __shared__ int s_rem;
  __shared__ typename FuseScan::TempStorage scan_tmp;
  const uint4* Ks = K + (static_cast<size_t>(slice) * T + t_lo) * 16;

  // ---- phase 1: token scores of [t_lo, t_hi) as orderable keys
  if (scorer == KVT_SCORER_KNORM) {
    for (int b0 = hw & ~1; b0 < n_loc; b0 += 16 * kFuseUnroll) {  // warp-uniform trip count
      uint4 v[kFuseUnroll];
#pragma unroll
      for (int u = 0; u < kFuseUnroll; ++u) {
        const int t = b0 + (hw & 1) + 16 * u;
        v[u] = t < n_loc ? Ks[static_cast<size_t>(t) * 16 + l16] : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kFuseUnroll; ++u) {
        const int t = b0 + (hw & 1) + 16 * u;
        const double n2 = half_butterfly(chunk_sumsq(v[u]));
        if (t < n_loc && l16 == 0) keys[t] = score_key(__double2float_rn(n2));
      }
    }
  } else {  // keydiff: exact fixed-point mean direction over the whole slice, then cosine
    long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int b0 = hw & ~1; b0 < n_loc; b0 += 16 * kFuseUnroll) {
      uint4 v[kFuseUnroll];
#pragma unroll
      for (int u = 0; u < kFuseUnroll; ++u) {
        const int t = b0 + (hw & 1) + 16 * u;
        v[u] = t < n_loc ? Ks[static_cast<size_t>(t) * 16 + l16] : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kFuseUnroll; ++u) {
        const double n2 = half_butterfly(chunk_sumsq(v[u]));
        const double inv = n2 > 0.0 ? __drcp_rn(__dsqrt_rn(n2)) : 0.0;
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double a = __dmul_rn(double(bf2f(w[j] & 0xffffu)), inv);
          const double b = __dmul_rn(double(bf2f(w[j] >> 16)), inv);
          acc[2 * j] += __double2ll_rn(__dmul_rn(a, kFx));
          acc[2 * j + 1] += __double2ll_rn(__dmul_rn(b, kFx));
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) part[hw][l16 * 8 + i] = acc[i];
    __syncthreads();
    if (tid < kD) {
      long long sum = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) sum += part[i][tid];
      sfix[tid] = sum;
    }
    cl.sync();
    if (tid < kD) {
      long long sum = 0;
      for (int c = 0; c < kFuseC; ++c) sum += cl.map_shared_rank(sfix, c)[tid];
      sdir[tid] = __dmul_rn(__ll2double_rn(sum), 1.0 / kFx);
    }
    __syncthreads();
    double sd[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) sd[i] = sdir[l16 * 8 + i];
    for (int b0 = hw & ~1; b0 < n_loc; b0 += 16 * kFuseUnroll) {
      uint4 v[kFuseUnroll];
#pragma unroll
      for (int u = 0; u < kFuseUnroll; ++u) {
        const int t = b0 + (hw & 1) + 16 * u;
        v[u] = t < n_loc ? Ks[static_cast<size_t>(t) * 16 + l16] : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kFuseUnroll; ++u) {
        const int t = b0 + (hw & 1) + 16 * u;
        const double n2 = half_butterfly(chunk_sumsq(v[u]));
        const double inv = n2 > 0.0 ? __drcp_rn(__dsqrt_rn(n2)) : 0.0;
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double x0 = __dmul_rn(double(bf2f(w[j] & 0xffffu)), inv);
          const double x1 = __dmul_rn(double(bf2f(w[j] >> 16)), inv);
          a = __dadd_rn(a, __dmul_rn(x0, sd[2 * j]));
          a = __dadd_rn(a, __dmul_rn(x1, sd[2 * j + 1]));
        }
        const double p = half_butterfly(a);
        if (t < n_loc && l16 == 0) keys[t] = score_key(__double2float_rn(-p));
      }
    }
  }
  __syncthreads();

  // ---- phase 2: cluster-wide MSB-first radix select of the k-th key
  uint32_t prefix = 0, mask = 0;
  int rem = k;
  for (int shift = 24, rd = 0; shift >= 0; shift -= 8, ++rd) {
    int* h = hist[rd & 1];
    h[tid] = 0;  // kFuseThreads == 256 bins
    __syncthreads();
    for (int t = tid; t < n_loc; t += kFuseThreads) {
      const uint32_t key = keys[t];
      if ((key & mask) == prefix) atomicAdd(&h[(key >> shift) & 255], 1);
    }
    cl.sync();
    {
      int sum = 0;
      for (int c = 0; c < kFuseC; ++c) sum += cl.map_shared_rank(h, c)[tid];
      tot[tid] = sum;
    }
    __syncthreads();
    if (tid == 0) {
      int b = 255;
      for (; b > 0; --b) {
        if (tot[b] >= rem) break;
        rem -= tot[b];
      }
      s_rem = rem;
      s_prefix = prefix | (uint32_t(b) << shift);
      s_mask = mask | (255u << shift);
    }
    __syncthreads();
    prefix = s_prefix;
    mask = s_mask;
    rem = s_rem;
  }
  const uint32_t kth = prefix;
  const int ties = rem;

  // ---- order-preserving compaction of the kept indices (ascending)
  const int seg = (n_loc + kFuseThreads - 1) / kFuseThreads;
  const int s0 = min(n_loc, tid * seg), s1 = min(n_loc, s0 + seg);
  int above = 0, eq = 0;
  for (int t = s0; t < s1; ++t) {
    const uint32_t key = keys[t];
    above += key > kth;
    eq += key == kth;
  }
  int above_before, eq_before, above_all, eq_all;
  FuseScan(scan_tmp).ExclusiveSum(above, above_before, above_all);
  __syncthreads();
  FuseScan(scan_tmp).ExclusiveSum(eq, eq_before, eq_all);
  if (tid == 0) {
    cnt[0] = above_all;
    cnt[1] = eq_all;
  }
  cl.sync();
  int a_base = 0, e_base = 0;
  for (int c = 0; c < rank; ++c) {
    const int* rc = cl.map_shared_rank(cnt, c);
    a_base += rc[0];
    e_base += rc[1];
  }
  int32_t* bidx = reinterpret_cast<int32_t*>(blob + m.idx_off);
  {
    int eq_seen = e_base + eq_before;
    int pos = a_base + above_before + min(eq_seen, ties);
    int32_t* out = bidx + static_cast<size_t>(slice) * k;
    for (int t = s0; t < s1; ++t) {
      const uint32_t key = keys[t];
      if (key > kth) {
        out[pos++] = t_lo + t;
      } else if (key == kth) {
        if (eq_seen < ties) out[pos++] = t_lo + t;
        ++eq_seen;
      }
    }
  }
  cl.sync();  // every CTA's indices are visible; no DSMEM access after this point

  // ---- phase 3: gather + quantise + pack (rows re-read from L2)
  if (bits == 16) {
    uint4* ko = reinterpret_cast<uint4*>(blob + m.kcode_off);
    uint4* vo = reinterpret_cast<uint4*>(blob + m.vcode_off);
    for (int jb = rank * 16; jb < k; jb += kFuseC * 16) {
      const int j = jb + hw;
      if (j < k) {
        const int t = bidx[static_cast<size_t>(slice) * k + j];
        const size_t src = (static_cast<size_t>(slice) * T + t) * 16 + l16;
        const size_t dst = (static_cast<size_t>(slice) * k + j) * 16 + l16;
        const uint4 a = __ldcs(K + src), b = __ldcs(V + src);
        __stcs(ko + dst, a);
        __stcs(vo + dst, b);
      }
    }
  } else {
    const int ng = (k + KVT_QGROUP - 1) / KVT_QGROUP;
    for (int g = rank; g < ng; g += kFuseC)
      pack_k_group(K, bidx, reinterpret_cast<uint32_t*>(blob + m.kcode_off),
                   reinterpret_cast<uint16_t*>(blob + m.kscale_off), reinterpret_cast<uint16_t*>(blob + m.kzero_off),
                   T, k, bits, slice, g, pk);
    for (int jb = rank * 16; jb < k; jb += kFuseC * 16)
      pack_v_row(V, bidx, nullptr, reinterpret_cast<uint32_t*>(blob + m.vcode_off),
                 reinterpret_cast<uint16_t*>(blob + m.vscale_off), reinterpret_cast<uint16_t*>(blob + m.vzero_off), T,
                 k, bits, slice, jb + hw);
  }
}

static bool fused_ok(const kvt_kv_shape* s, const kvt_codec_cfg* c) {
  return c->scorer != KVT_SCORER_SNAPKV && fuse_smem_bytes(s->T) <= kFuseMaxSmem;
}

static int launch_fused(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k,
                        const uint16_t* v, void* blob) {
  kvt_blob_map m;
  blob_map(*s, *c, &m);
  const size_t smem = fuse_smem_bytes(s->T);
  static bool attr = false;
  if (!attr) {
    KVT_CUDA_TRY(cudaFuncSetAttribute(k_compress_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFuseMaxSmem)));
    attr = true;
  }
  dim3 grid(kFuseC, s->L * s->H);
  k_compress_fused<<<grid, kFuseThreads, smem, h->stream>>>(reinterpret_cast<const uint4*>(k),
                                                             reinterpret_cast<const uint4*>(v), s->T, c->keep, c->bits,
                                                             c->scorer, m, static_cast<char*>(blob));
  LAUNCHED(h);
  return KVT_OK;
}

// ---------------------------------------------------------------- compress

extern "C" int kvt_compress(kvt_handle* h, const kvt_kv_shape* s, const kvt_codec_cfg* c, const uint16_t* k,
                            const uint16_t* v, void* workspace, void* blob) {
  int rc;
  if ((rc = check_shape(s, c))) return rc;
  if (fused_ok(s, c) && !getenv("KVT_UNFUSED")) return launch_fused(h, s, c, k, v, blob);
  char* w = static_cast<char*>(workspace);
  float* scores = reinterpret_cast<float*>(w);
  float* votes = reinterpret_cast<float*>(w + ws_scores(s));
  auto* fixed = reinterpret_cast<unsigned long long*>(w + 2 * ws_scores(s));
  int32_t* idx = reinterpret_cast<int32_t*>(w + 2 * ws_scores(s) + ws_fixed(s));
  if ((rc = launch_scores(h, s, c, k, scores, votes, fixed))) return rc;
  if ((rc = launch_topk(h, s, c, scores, idx))) return rc;
  return launch_pack(h, s, c, k, v, idx, blob);
}
