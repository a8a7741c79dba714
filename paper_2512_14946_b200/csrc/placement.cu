// Placement hot path on sm_100a: candidate scoring (K1, fused best_config)
// and the least-utility-drop greedy (K2 per-resident best update + K3
// persistent single-warp resolver) behind the kvt_* C ABI.
//
// Reference: proj/src/utility.cpp (scoring), proj/src/placement.cpp (store +
// greedy). Results are bit-identical to the reference library (tests/).
//
// Greedy design. A resident's update options depend only on
// its own (tier, config, profile) (utility.cpp:81-127), so each resident
// caches its best option key (drop, bytes_freed, enumeration index) and a
// per-tier 32-ary tournament tree keeps the tier-wide argmin under the
// reference's total order (drop asc, bytes_freed desc, context asc;
// placement.cpp:165-170). One step = read root, apply, recompute one
// resident with one warp, update <= 2 tree paths of depth log32(N). The
// whole insert/resolve sequence runs in ONE persistent warp: the
// dependency chain is strictly sequential, so the kernel is built for
// latency (no block barriers, no host round trips between steps).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <memory>
#include <limits>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>


#include "kvt_common.cuh"

namespace kvt {

static thread_local std::string g_err;

int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace {
std::mutex g_dev_mu;
std::map<int, std::pair<int, int>> g_dev_info;  // device -> (SMs, smem opt-in)
std::map<std::tuple<const void*, int, int>, int> g_attr;  // (fn, device, attribute) -> value set
std::map<std::tuple<const void*, int, long long>, int> g_cached;

const std::pair<int, int>& dev_info(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_dev_info.find(dev);
  if (it == g_dev_info.end()) {
    int sms = 0, optin = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    it = g_dev_info.emplace(dev, std::make_pair(sms > 0 ? sms : 148, optin > 0 ? optin : 232448)).first;
  }
  return it->second;
}
}  // namespace

int device_sms(int dev) { return dev_info(dev).first; }
int device_smem_optin(int dev) { return dev_info(dev).second; }

cudaError_t func_attr(const void* fn, int dev, cudaFuncAttribute a, int value) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  const auto key = std::make_tuple(fn, dev, static_cast<int>(a));
  auto it = g_attr.find(key);
  if (it != g_attr.end() && it->second == value) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, a, value);
  if (e == cudaSuccess) g_attr[key] = value;
  return e;
}

int cached_per_device(const void* fn, int dev, long long key, int (*compute)(void*), void* arg) {
  const auto k = std::make_tuple(fn, dev, key);
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_cached.find(k);
    if (it != g_cached.end()) return it->second;
  }
  const int v = compute(arg);  // outside the lock: may call into the driver
  std::lock_guard<std::mutex> lk(g_dev_mu);
  return g_cached.emplace(k, v).first->second;
}

}  // namespace kvt

using namespace kvt;



extern "C" const char* kvt_last_error(void) { return g_err.c_str(); }
extern "C" int kvt_abi_version(void) { return KVT_ABI_VERSION; }

static int ensure_scratch(kvt_handle* h, size_t bytes) {
  if (h->scratch_bytes >= bytes) return KVT_OK;
  if (h->scratch) cudaFree(h->scratch);
  h->scratch = nullptr;
  h->scratch_bytes = 0;
  KVT_CUDA_TRY(cudaMalloc(&h->scratch, bytes));
  h->scratch_bytes = bytes;
  return KVT_OK;
}

extern "C" int kvt_create(int device, void* stream, kvt_handle** out) {
  if (!out) return set_error(KVT_EINVAL, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return set_error(KVT_ECUDA, std::string("no CUDA device visible: ") + cudaGetErrorString(e));
  if (device < 0 || device >= n) return set_error(KVT_EINVAL, "device ordinal out of range");
  DeviceGuard dg(device);
  cudaDeviceProp prop;
  KVT_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return set_error(KVT_ECUDA, std::string("libkvt_b200 is built for sm_100a, device is ") + prop.name);
  auto* h = new kvt_handle();
  h->device = device;
  h->stream = static_cast<cudaStream_t>(stream);
  *out = h;
  return KVT_OK;
}

kvt_handle::~kvt_handle() {
  DeviceGuard dg(device);
  if (scratch) cudaFree(scratch);
  if (snapq) cudaFree(snapq);
  if (snape) cudaFree(snape);
  for (int i = 0; i < 4; ++i) {
    if (move_s[i]) cudaStreamSynchronize(move_s[i]), cudaStreamDestroy(move_s[i]);
    if (move_done[i]) cudaEventDestroy(move_done[i]);
  }
  if (move_start) cudaEventDestroy(move_start);
}

extern "C" int kvt_destroy(kvt_handle* h) {
  delete h;  // frees scratch, snapkv caches and the tier-move streams / events
  return KVT_OK;
}

extern "C" int kvt_sync(kvt_handle* h) {
  KVT_ON_DEVICE(h);
  KVT_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return KVT_OK;
}

extern "C" int kvt_set_stream(kvt_handle* h, void* stream) {
  h->stream = static_cast<cudaStream_t>(stream);
  return KVT_OK;
}

extern "C" int64_t kvt_launch_count(kvt_handle* h) { return h->launches; }

// ------------------------------------------------------------ host resolve

// CandidateSpace ctor proj/src/utility.cpp:21-33, MethodSet ctor
// proj/src/core.cpp:10-27.
static int resolve_space(const kvt_space* sp, DevSpace* s) {
  if (!sp) return set_error(KVT_EINVAL, "null space");
  if (sp->n_methods <= 0) return set_error(KVT_EVALIDATION, "method set must not be empty");
  if (sp->n_methods > KVT_MAX_METHODS) return set_error(KVT_EINVAL, "too many methods for the device kernels");
  if (sp->n_ratios <= 0) return set_error(KVT_EVALIDATION, "candidate ratio grid must not be empty");
  if (sp->n_ratios > KVT_MAX_RATIOS) return set_error(KVT_EINVAL, "too many ratios for the device kernels");
  std::memset(s, 0, sizeof(*s));
  s->M = sp->n_methods;
  for (int m = 0; m < s->M; ++m) {
    const char* nm = sp->method_names[m];
    if (!nm || !nm[0]) return set_error(KVT_EVALIDATION, "compression method name must not be empty");
    for (int j = 0; j < m; ++j)
      if (std::strcmp(sp->method_names[j], nm) == 0)
        return set_error(KVT_EVALIDATION, std::string("duplicate compression method name: ") + nm);
    if (sp->decompression_overhead[m] < 0.0)
      return set_error(KVT_EVALIDATION, std::string("negative decompression overhead for method ") + nm);
    s->ovh[m] = sp->decompression_overhead[m];
  }
  for (int m = 0; m < s->M; ++m) {  // byte-lexicographic rank (std::string operator<)
    int rank = 0;
    for (int j = 0; j < s->M; ++j)
      if (std::strcmp(sp->method_names[j], sp->method_names[m]) < 0) ++rank;
    s->name_rank[m] = rank;
  }
  std::vector<double> r(sp->ratios, sp->ratios + sp->n_ratios);
  for (double v : r)
    if (!(v > 0.0) || v > 1.0 || !std::isfinite(v))
      return set_error(KVT_EVALIDATION, "candidate ratio out of (0, 1]");
  std::sort(r.begin(), r.end(), [](double a, double b) { return a > b; });
  r.erase(std::unique(r.begin(), r.end()), r.end());
  s->R = static_cast<int>(r.size());
  for (int i = 0; i < s->R; ++i) s->ratio[i] = r[i];
  return KVT_OK;
}

// validate_hierarchy proj/src/core.cpp:86-121
static int resolve_tiers(const kvt_tier* in, int n, DevTiers* o) {
  if (n <= 0) return set_error(KVT_EVALIDATION, "hierarchy must have at least one tier");
  if (n > KVT_MAX_TIERS) return set_error(KVT_EINVAL, "too many tiers for the device kernels");
  std::vector<kvt_tier> t(in, in + n);
  std::stable_sort(t.begin(), t.end(), [](const kvt_tier& a, const kvt_tier& b) { return a.tier_id < b.tier_id; });
  std::memset(o, 0, sizeof(*o));
  o->T = n;
  for (int i = 0; i < n; ++i) {
    const std::string tid = std::to_string(t[i].tier_id);
    if (i + 1 < n && t[i + 1].tier_id == t[i].tier_id)
      return set_error(KVT_EVALIDATION, "duplicate tier_id " + tid);
    if (t[i].unlimited && i + 1 != n)
      return set_error(KVT_EVALIDATION, "unlimited capacity is only allowed on the bottom tier (tier " + tid + ")");
    if (!t[i].unlimited && t[i].capacity_bytes < 0)
      return set_error(KVT_EVALIDATION, "negative capacity on tier " + tid);
    if (!(t[i].read_bandwidth > 0.0) || !std::isfinite(t[i].read_bandwidth))
      return set_error(KVT_EVALIDATION, "read bandwidth must be > 0 on tier " + tid);
    if (t[i].fixed_access_latency < 0.0 || !std::isfinite(t[i].fixed_access_latency))
      return set_error(KVT_EVALIDATION, "fixed access latency must be >= 0 on tier " + tid);
    o->id[i] = t[i].tier_id;
    o->unlimited[i] = t[i].unlimited ? 1 : 0;
    o->cap[i] = t[i].capacity_bytes;
    o->bw[i] = t[i].read_bandwidth;
    o->lat[i] = t[i].fixed_access_latency;
  }
  return KVT_OK;
}

static uint64_t fnv(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// ----------------------------------------------------------------- profiles

struct kvt_pset {
  kvt_handle* h = nullptr;
  DevProfiles dev{};
  void* buf = nullptr;
  uint64_t id = 0;
};

static std::atomic<uint64_t> g_pset_counter{0};

extern "C" int kvt_pset_create(kvt_handle* h, const kvt_profiles* pr, kvt_pset** out) {
  KVT_ON_DEVICE(h);
  if (!h || !pr || !out) return set_error(KVT_EINVAL, "null argument");
  if (pr->n_ctx < 0 || pr->n_methods <= 0 || pr->n_methods > KVT_MAX_METHODS)
    return set_error(KVT_EINVAL, "bad profile set dimensions");
  const int n = pr->n_ctx, M = pr->n_methods;
  const int G = pr->grid_offset[n];
  for (int c = 0; c < n; ++c) {
    if (pr->grid_offset[c + 1] <= pr->grid_offset[c])
      return set_error(KVT_EVALIDATION, "profile ratio grid is empty for context " + std::to_string(c));
    if (pr->original_size_bytes[c] <= 0)
      return set_error(KVT_EVALIDATION, "original size must be > 0");
  }
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_orig = 0;
  const size_t o_freq = o_orig + align(sizeof(long long) * (n + 1));
  const size_t o_goff = o_freq + align(sizeof(double) * (n + 1));
  const size_t o_grid = o_goff + align(sizeof(int) * (n + 1));
  const size_t o_qual = o_grid + align(sizeof(double) * (G + 1));
  const size_t o_has = o_qual + align(sizeof(double) * (static_cast<size_t>(G) * M + 1));
  const size_t total = o_has + align(static_cast<size_t>(n) * M + 1);
  auto* p = new kvt_pset();
  p->h = h;
  cudaError_t e = cudaMalloc(&p->buf, total);
  if (e != cudaSuccess) {
    delete p;
    return set_error(KVT_ECUDA, std::string("cudaMalloc profiles: ") + cudaGetErrorString(e));
  }
  char* b = static_cast<char*>(p->buf);
  cudaStream_t s = h->stream;
  cudaMemcpyAsync(b + o_orig, pr->original_size_bytes, sizeof(long long) * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(b + o_freq, pr->frequency, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(b + o_goff, pr->grid_offset, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(b + o_grid, pr->grid, sizeof(double) * G, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(b + o_qual, pr->quality, sizeof(double) * static_cast<size_t>(G) * M, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(b + o_has, pr->has_method, static_cast<size_t>(n) * M, cudaMemcpyHostToDevice, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFree(p->buf);
    delete p;
    return set_error(KVT_ECUDA, std::string("profile upload: ") + cudaGetErrorString(e));
  }
  p->dev.n = n;
  p->dev.M = M;
  p->dev.orig = reinterpret_cast<const long long*>(b + o_orig);
  p->dev.freq = reinterpret_cast<const double*>(b + o_freq);
  p->dev.goff = reinterpret_cast<const int*>(b + o_goff);
  p->dev.grid = reinterpret_cast<const double*>(b + o_grid);
  p->dev.qual = reinterpret_cast<const double*>(b + o_qual);
  p->dev.has = reinterpret_cast<const unsigned char*>(b + o_has);
  p->id = ++g_pset_counter;
  *out = p;
  return KVT_OK;
}

// ---------------------------------------------- multi-GPU profile exchange
// include/kvt_b200.h "record": one rank's profile rows as a flat byte record
// (NCCL all-gathers equal-sized records); kvt_pset_merge concatenates the
// gathered records in rank order on the device and rebases grid offsets.
namespace kvt_rec {  // named: kernel parameter types cannot live in an anonymous namespace
struct RecLayout {
  int64_t orig, freq, grid, qual, goff, has, total;
};
int64_t rec_al(int64_t x) { return (x + 255) & ~int64_t(255); }
RecLayout rec_layout(int64_t n, int64_t g, int64_t M) {
  RecLayout L;
  L.orig = 0;
  L.freq = L.orig + rec_al(8 * n);
  L.grid = L.freq + rec_al(8 * n);
  L.qual = L.grid + rec_al(8 * g);
  L.goff = L.qual + rec_al(8 * g * M);
  L.has = L.goff + rec_al(4 * (n + 1));
  L.total = L.has + rec_al(n * M);
  return L;
}
// pset buffer sections (same layout as kvt_pset_create)
struct PsetLayout {
  size_t orig, freq, goff, grid, qual, has, total;
};
PsetLayout pset_layout(size_t n, size_t G, size_t M) {
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  PsetLayout P;
  P.orig = 0;
  P.freq = P.orig + align(sizeof(long long) * (n + 1));
  P.goff = P.freq + align(sizeof(double) * (n + 1));
  P.grid = P.goff + align(sizeof(int) * (n + 1));
  P.qual = P.grid + align(sizeof(double) * (G + 1));
  P.has = P.qual + align(sizeof(double) * (G * M + 1));
  P.total = P.has + align(n * M + 1);
  return P;
}
}  // namespace kvt_rec
using namespace kvt_rec;

// One block-row per (rank, section): 8-byte (or 1-byte for has) grid-stride
// copies of the record sections into the global arrays, goff rebased.
__global__ void __launch_bounds__(256) k_pset_merge(const uint8_t* __restrict__ rec, RecLayout L, int n, int g, int M,
                                                    char* __restrict__ dst, PsetLayout P) {
  const int r = blockIdx.y, sec = blockIdx.z;
  const uint8_t* b = rec + static_cast<size_t>(r) * L.total;
  const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x, step = size_t(gridDim.x) * blockDim.x;
  auto copy8 = [&](int64_t src_off, size_t dst_off, size_t n8) {
    const unsigned long long* s = reinterpret_cast<const unsigned long long*>(b + src_off);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(dst + dst_off);
    for (size_t i = tid; i < n8; i += step) d[i] = s[i];
  };
  switch (sec) {
    case 0: copy8(L.orig, P.orig + 8 * size_t(r) * n, n); break;
    case 1: copy8(L.freq, P.freq + 8 * size_t(r) * n, n); break;
    case 2: copy8(L.grid, P.grid + 8 * size_t(r) * g, g); break;
    case 3: copy8(L.qual, P.qual + 8 * size_t(r) * g * M, size_t(g) * M); break;
    case 4: {
      const int* s = reinterpret_cast<const int*>(b + L.goff);
      int* d = reinterpret_cast<int*>(dst + P.goff) + size_t(r) * n;
      for (size_t i = tid; i < size_t(n); i += step) d[i] = r * g + s[i];
      if (r == gridDim.y - 1 && tid == 0) d[n] = (r + 1) * g;  // goff[world * n] = world * g
      break;
    }
    default: {
      const uint8_t* s = b + L.has;
      uint8_t* d = reinterpret_cast<uint8_t*>(dst + P.has) + size_t(r) * n * M;
      for (size_t i = tid; i < size_t(n) * M; i += step) d[i] = s[i];
    }
  }
}

extern "C" int64_t kvt_pset_record_bytes(int32_t n_ctx, int32_t grid_len, int32_t n_methods) {
  return rec_layout(n_ctx, grid_len, n_methods).total;
}

extern "C" int kvt_pset_record_pack(const kvt_profiles* pr, void* record) {
  if (!pr || !record || pr->n_ctx < 0 || pr->n_methods <= 0 || pr->n_methods > KVT_MAX_METHODS)
    return set_error(KVT_EINVAL, "bad profile set dimensions");
  const int n = pr->n_ctx, M = pr->n_methods, g = pr->grid_offset[n];
  for (int c = 0; c < n; ++c) {
    if (pr->grid_offset[c + 1] <= pr->grid_offset[c])
      return set_error(KVT_EVALIDATION, "profile ratio grid is empty for context " + std::to_string(c));
    if (pr->original_size_bytes[c] <= 0) return set_error(KVT_EVALIDATION, "original size must be > 0");
  }
  const RecLayout L = rec_layout(n, g, M);
  char* b = static_cast<char*>(record);
  std::memset(b, 0, static_cast<size_t>(L.total));
  std::memcpy(b + L.orig, pr->original_size_bytes, 8 * size_t(n));
  std::memcpy(b + L.freq, pr->frequency, 8 * size_t(n));
  std::memcpy(b + L.grid, pr->grid, 8 * size_t(g));
  std::memcpy(b + L.qual, pr->quality, 8 * size_t(g) * M);
  std::memcpy(b + L.goff, pr->grid_offset, 4 * size_t(n + 1));
  std::memcpy(b + L.has, pr->has_method, size_t(n) * M);
  return KVT_OK;
}

extern "C" int kvt_pset_merge(kvt_handle* h, const void* records, int32_t world, int32_t n_ctx, int32_t grid_len,
                              int32_t n_methods, kvt_pset** out) {
  KVT_ON_DEVICE(h);
  if (!records || !out || world < 1 || n_ctx < 0 || grid_len < 0 || n_methods <= 0 || n_methods > KVT_MAX_METHODS)
    return set_error(KVT_EINVAL, "bad merge request");
  const size_t N = size_t(world) * n_ctx, G = size_t(world) * grid_len, M = n_methods;
  const PsetLayout P = pset_layout(N, G, M);
  kvt_pset* p = *out;
  if (p && (p->dev.n != static_cast<int>(N) || p->dev.M != n_methods || p->h != h))
    return set_error(KVT_EINVAL, "kvt_pset_merge: the set to refill has other dimensions");
  if (!p) {
    p = new kvt_pset();
    p->h = h;
    cudaError_t e = cudaMalloc(&p->buf, P.total);
    if (e != cudaSuccess) {
      delete p;
      return set_error(KVT_ECUDA, std::string("cudaMalloc profiles: ") + cudaGetErrorString(e));
    }
    char* b = static_cast<char*>(p->buf);
    p->dev.n = static_cast<int>(N);
    p->dev.M = n_methods;
    p->dev.orig = reinterpret_cast<const long long*>(b + P.orig);
    p->dev.freq = reinterpret_cast<const double*>(b + P.freq);
    p->dev.goff = reinterpret_cast<const int*>(b + P.goff);
    p->dev.grid = reinterpret_cast<const double*>(b + P.grid);
    p->dev.qual = reinterpret_cast<const double*>(b + P.qual);
    p->dev.has = reinterpret_cast<const unsigned char*>(b + P.has);
  }
  const RecLayout L = rec_layout(n_ctx, grid_len, n_methods);
  const int bx = static_cast<int>(std::min<size_t>(64, (std::max<size_t>(size_t(grid_len) * M, n_ctx) + 255) / 256 + 1));
  k_pset_merge<<<dim3(bx, world, 6), 256, 0, h->stream>>>(static_cast<const uint8_t*>(records), L, n_ctx, grid_len,
                                                           n_methods, static_cast<char*>(p->buf), P);
  h->launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (!*out) {
      cudaFree(p->buf);
      delete p;
    }
    return set_error(KVT_ECUDA, std::string("k_pset_merge: ") + cudaGetErrorString(e));
  }
  p->id = ++g_pset_counter;  // new contents: scoring caches keyed by the set id refresh
  *out = p;
  return KVT_OK;
}

extern "C" int kvt_pset_destroy(kvt_pset* p) {
  KVT_ON_DEVICE((p ? p->h : nullptr));
  if (!p) return KVT_OK;
  cudaFree(p->buf);
  delete p;
  return KVT_OK;
}

// ------------------------------------------------------------- K1 scoring

struct Tables {  // dense candidate tables, see include/kvt_b200.h
  long long* size;      // [n][R]
  double* q;            // [n][M][R]
  unsigned char* valid; // [n][M][R]
  double* ttft;         // [n][T][M][R] (nullable)
  double* u;            // [n][T][M][R]
  kvt_best* best;       // [n] (nullable)
};

// candidate_preferred proj/src/utility.cpp:147-157; j = enumeration index
struct CandKey {
  double u, q, ratio;
  int tier_id, name_rank, j;
};

__device__ __forceinline__ bool cand_better(const CandKey& a, const CandKey& b, int rule) {
  if (a.j < 0) return false;
  if (b.j < 0) return true;
  if (rule == KVT_RULE_QUALITY_FIRST && a.q != b.q) return a.q > b.q;
  if (a.u != b.u) return a.u > b.u;
  if (a.q != b.q) return a.q > b.q;
  if (a.tier_id != b.tier_id) return a.tier_id < b.tier_id;
  if (a.ratio != b.ratio) return a.ratio > b.ratio;
  if (a.name_rank != b.name_rank) return a.name_rank < b.name_rank;
  return a.j < b.j;  // first enumerated wins exact ties (utility.cpp:167-170)
}

__device__ __forceinline__ CandKey shfl_cand(const CandKey& k, int lane_mask) {
  CandKey o;
  o.u = __shfl_xor_sync(0xffffffffu, k.u, lane_mask);
  o.q = __shfl_xor_sync(0xffffffffu, k.q, lane_mask);
  o.ratio = __shfl_xor_sync(0xffffffffu, k.ratio, lane_mask);
  o.tier_id = __shfl_xor_sync(0xffffffffu, k.tier_id, lane_mask);
  o.name_rank = __shfl_xor_sync(0xffffffffu, k.name_rank, lane_mask);
  o.j = __shfl_xor_sync(0xffffffffu, k.j, lane_mask);
  return o;
}

constexpr int kScoreWarps = 4;

// One warp per context: quality_of per (method, ratio) once, then the
// tier x method x ratio cross product (all_candidates order, utility.cpp:
// 129-145) with the best_config argmax fused in.
__global__ void __launch_bounds__(kScoreWarps * 32)
k_score(DevProfiles P, DevSpace S, DevTiers TT, double alpha, int rule, Tables out) {
  __shared__ double sq[kScoreWarps][KVT_MAX_METHODS * KVT_MAX_RATIOS];
  __shared__ unsigned char sv[kScoreWarps][KVT_MAX_METHODS * KVT_MAX_RATIOS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kScoreWarps + warp;
  if (c >= P.n) return;
  const int M = S.M, R = S.R, T = TT.T, MR = M * R;
  const long long orig = P.orig[c];
  const double f = P.freq[c];
  for (int k = lane; k < MR; k += 32) {
    const int m = k / R, r = k - m * R;
    const double ratio = S.ratio[r];
    double q = 0.0;
    bool ok = scorable(P, c, m, ratio);
    if (ok) ok = quality_of(P, c, m, ratio, &q);
    sq[warp][k] = ok ? q : 0.0;
    sv[warp][k] = ok ? 1 : 0;
    out.q[static_cast<size_t>(c) * MR + k] = ok ? q : 0.0;
    out.valid[static_cast<size_t>(c) * MR + k] = ok ? 1 : 0;
  }
  for (int r = lane; r < R; r += 32) out.size[static_cast<size_t>(c) * R + r] = csize(orig, S.ratio[r]);
  __syncwarp();
  CandKey best;
  best.j = -1;
  best.u = best.q = best.ratio = 0.0;
  best.tier_id = best.name_rank = 0;
  const size_t ubase = static_cast<size_t>(c) * T * MR;
  for (int j = lane; j < T * MR; j += 32) {
    const int t = j / MR, k = j - t * MR;
    const int m = k / R, r = k - m * R;
    if (!sv[warp][k]) {
      out.u[ubase + j] = 0.0;
      if (out.ttft) out.ttft[ubase + j] = 0.0;
      continue;
    }
    const long long sz = csize(orig, S.ratio[r]);
    const double tt = load_time(sz, TT.lat[t], TT.bw[t], S.ovh[m]);
    const double u = utility_score(sq[warp][k], tt, f, alpha);
    out.u[ubase + j] = u;
    if (out.ttft) out.ttft[ubase + j] = tt;
    CandKey cand{u, sq[warp][k], S.ratio[r], TT.id[t], S.name_rank[m], j};
    if (cand_better(cand, best, rule)) best = cand;
  }
  if (!out.best) return;
  for (int off = 16; off > 0; off >>= 1) {
    CandKey o = shfl_cand(best, off);
    if (cand_better(o, best, rule)) best = o;
  }
  if (lane == 0) {
    kvt_best b = {};
    if (best.j < 0) {
      b.status = 1;
    } else {
      const int t = best.j / MR, k = best.j - t * MR;
      const int m = k / R, r = k - m * R;
      b.tier_index = t;
      b.tier_id = TT.id[t];
      b.method = m;
      b.ratio_index = r;
      b.ratio = S.ratio[r];
      b.size_bytes = csize(orig, S.ratio[r]);
      b.quality = best.q;
      b.ttft = load_time(b.size_bytes, TT.lat[t], TT.bw[t], S.ovh[m]);
      b.utility = best.u;
    }
    out.best[c] = b;
  }
}

static int launch_score(kvt_handle* h, const DevProfiles& P, const DevSpace& S, const DevTiers& T,
                        double alpha, int rule, const Tables& out) {
  if (P.n == 0) return KVT_OK;
  const int blocks = (P.n + kScoreWarps - 1) / kScoreWarps;
  k_score<<<blocks, kScoreWarps * 32, 0, h->stream>>>(P, S, T, alpha, rule, out);
  h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  return KVT_OK;
}

extern "C" int kvt_score_candidates(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, int32_t n_tiers,
                                    const kvt_space* space, const kvt_params* params, int64_t* size,
                                    double* quality, uint8_t* valid, double* ttft, double* utility) {
  KVT_ON_DEVICE(h);
  DevSpace S;
  DevTiers T;
  int rc;
  if ((rc = resolve_space(space, &S))) return rc;
  if ((rc = resolve_tiers(tiers, n_tiers, &T))) return rc;
  if (p->dev.M != S.M) return set_error(KVT_EINVAL, "profile set / space method count mismatch");
  const size_t n = p->dev.n, R = S.R, MR = S.M * S.R, TMR = T.T * MR;
  const size_t b_size = n * R * 8, b_q = n * MR * 8, b_v = (n * MR + 255) & ~size_t(255), b_u = n * TMR * 8;
  if ((rc = ensure_scratch(h, b_size + b_q + b_v + 2 * b_u + 1024))) return rc;
  char* b = static_cast<char*>(h->scratch);
  Tables t{reinterpret_cast<long long*>(b), reinterpret_cast<double*>(b + b_size),
           reinterpret_cast<unsigned char*>(b + b_size + b_q),
           reinterpret_cast<double*>(b + b_size + b_q + b_v),
           reinterpret_cast<double*>(b + b_size + b_q + b_v + b_u), nullptr};
  if ((rc = launch_score(h, p->dev, S, T, params->alpha, KVT_RULE_UTILITY, t))) return rc;
  cudaStream_t s = h->stream;
  if (size) KVT_CUDA_TRY(cudaMemcpyAsync(size, t.size, b_size, cudaMemcpyDeviceToHost, s));
  if (quality) KVT_CUDA_TRY(cudaMemcpyAsync(quality, t.q, b_q, cudaMemcpyDeviceToHost, s));
  if (valid) KVT_CUDA_TRY(cudaMemcpyAsync(valid, t.valid, n * MR, cudaMemcpyDeviceToHost, s));
  if (ttft) KVT_CUDA_TRY(cudaMemcpyAsync(ttft, t.ttft, b_u, cudaMemcpyDeviceToHost, s));
  if (utility) KVT_CUDA_TRY(cudaMemcpyAsync(utility, t.u, b_u, cudaMemcpyDeviceToHost, s));
  KVT_CUDA_TRY(cudaStreamSynchronize(s));
  return KVT_OK;
}

static int num_sms_p() {
  int dev = 0;
  cudaGetDevice(&dev);
  return device_sms(dev);
}

// ---------------------------------------------------------------- oracle_mckp
// proj/src/placement.cpp:300-372. Every context's scorable candidates in
// candidate_preferred order (stable over the enumeration order); a branch
// and bound over one-candidate-per-context assignments under the finite
// tiers' capacities. The first d contexts' choices index the GPU threads
// (mixed radix, context 0 most significant = the DFS's lexicographic
// order); persistent threads take the prefixes from a counter and run the reference's DFS on each
// subtree. A thread keeps the first maximal leaf of its subtree (strictly
// better only), so the maximal total with the smallest prefix index, then
// the thread's pick, is the reference's result: the first optimum in DFS
// order. Pruning: the reference's own test within a thread (bound <= its
// best), and a strict test against the best total any thread has reached
// (never cuts a subtree that could tie), shared as an order-preserving key.
// Per-thread DFS state lives in fixed arrays: 24 contexts (registers /
// L1-resident local memory) or 256 (an instance with more than 24 contexts
// passes the reference's max_assignments guard only when most of its
// contexts have a single candidate; those are forced levels of the same DFS).
constexpr int kMckpSmallCtx = 24;
constexpr int kMckpMaxCtx = 256;

__device__ __forceinline__ unsigned long long mckp_key(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(v, 0.0)));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double mckp_val(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

template <int NMAX>
__global__ void __launch_bounds__(128) k_mckp(const double* __restrict__ cu, const long long* __restrict__ csz,
                                              const int* __restrict__ ctier, const int* __restrict__ off,
                                              const int* __restrict__ cnt, const double* __restrict__ suffix,
                                              DevTiers TT, int n, int d, long long nprefix,
                                              unsigned long long* __restrict__ gbest,
                                              unsigned long long* __restrict__ next, double* __restrict__ out_total,
                                              int* __restrict__ out_found, long long* __restrict__ out_pfx,
                                              int* __restrict__ out_choice) {
  // persistent threads take prefixes from a counter (in increasing order per
  // thread, so a thread's first maximal leaf is its lexicographically first)
  const long long me = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  int choice[NMAX], k[NMAX], best_choice[NMAX];
  double tot[NMAX + 1];
  long long used[KVT_MAX_TIERS];
  double best = 0.0;
  long long best_pfx = -1;
  bool found = false;
  while (true) {
    const long long pfx = static_cast<long long>(atomicAdd(next, 1ull));
    if (pfx >= nprefix) break;
    for (int t = 0; t < KVT_MAX_TIERS; ++t) used[t] = 0;
    long long rem = pfx;
    for (int i = d - 1; i >= 0; --i) {
      choice[i] = static_cast<int>(rem % cnt[i]);
      rem /= cnt[i];
    }
    tot[0] = 0.0;
    bool fits = true;
    for (int i = 0; i < d && fits; ++i) {  // the prefix: the same capacity test and running sum as the DFS
      const int c = off[i] + choice[i], t = ctier[c];
      if (!TT.unlimited[t] && used[t] + csz[c] > TT.cap[t]) {
        fits = false;
        break;
      }
      used[t] += csz[c];
      tot[i + 1] = __dadd_rn(tot[i], cu[c]);
    }
    if (!fits) continue;
    int lvl = d;
    bool enter = true;
    while (true) {
      if (enter) {  // node entry (the reference's dfs(i, total) prologue)
        const double bound = __dadd_rn(tot[lvl], suffix[lvl]);
        if ((found && bound <= best) || bound < mckp_val(*const_cast<volatile unsigned long long*>(gbest))) {
          enter = false;  // pruned: back to the parent
        } else if (lvl == n) {
          best = tot[n];
          found = true;
          best_pfx = pfx;
          for (int i = 0; i < n; ++i) best_choice[i] = choice[i];
          atomicMax(gbest, mckp_key(best));
          enter = false;
        } else {
          k[lvl] = 0;
          enter = false;
          goto try_children;
        }
        if (lvl == d) break;
        --lvl;
        {
          const int c = off[lvl] + choice[lvl];
          used[ctier[c]] -= csz[c];
        }
        ++k[lvl];
      }
    try_children:
      while (k[lvl] < cnt[lvl]) {
        const int c = off[lvl] + k[lvl], t = ctier[c];
        if (!TT.unlimited[t] && used[t] + csz[c] > TT.cap[t]) {
          ++k[lvl];
          continue;
        }
        used[t] += csz[c];
        choice[lvl] = k[lvl];
        tot[lvl + 1] = __dadd_rn(tot[lvl], cu[c]);
        ++lvl;
        enter = true;
        break;
      }
      if (enter) continue;
      if (lvl == d) break;
      --lvl;
      {
        const int c = off[lvl] + choice[lvl];
        used[ctier[c]] -= csz[c];
      }
      ++k[lvl];
    }
  }
  out_found[me] = found ? 1 : 0;
  if (found) {
    out_total[me] = best;
    out_pfx[me] = best_pfx;
    for (int i = 0; i < n; ++i) out_choice[me * n + i] = best_choice[i];
  }
}

// the winning subtree: maximal total, then the smallest prefix index
__global__ void __launch_bounds__(1024) k_mckp_pick(const double* __restrict__ tot, const int* __restrict__ found,
                                                     const long long* __restrict__ pfx, long long nprefix,
                                                     long long* __restrict__ win) {
  __shared__ double sv[1024];
  __shared__ long long si[1024];
  const int tid = threadIdx.x;
  double bv = 0.0;
  long long bi = -1;
  for (long long i = tid; i < nprefix; i += 1024)  // (here: one entry per search thread)
    if (found[i] && (bi < 0 || tot[i] > bv || (tot[i] == bv && pfx[i] < pfx[bi]))) {
      bv = tot[i];
      bi = i;
    }
  sv[tid] = bv;
  si[tid] = bi;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (tid < w) {
      const double ov = sv[tid + w];
      const long long oi = si[tid + w];
      if (oi >= 0 && (si[tid] < 0 || ov > sv[tid] || (ov == sv[tid] && pfx[oi] < pfx[si[tid]]))) {
        sv[tid] = ov;
        si[tid] = oi;
      }
    }
    __syncthreads();
  }
  if (tid == 0) *win = si[0];
}

extern "C" int kvt_oracle_mckp(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, int32_t n_tiers,
                               const kvt_space* space, const kvt_params* params, double max_assignments,
                               double* total_utility, kvt_best* out) {
  KVT_ON_DEVICE(h);
  DevSpace S;
  DevTiers T;
  int rc;
  if ((rc = resolve_space(space, &S))) return rc;
  if ((rc = resolve_tiers(tiers, n_tiers, &T))) return rc;
  if (p->dev.M != S.M) return set_error(KVT_EINVAL, "profile set / space method count mismatch");
  const int n = p->dev.n, M = S.M, R = S.R, TT = T.T, MR = M * R;
  if (n > kMckpMaxCtx)
    return set_error(KVT_EVALIDATION, "instance too large for the exact solver: more than " +
                                          std::to_string(kMckpMaxCtx) + " contexts");
  // K1 candidate tables for every (context, tier, method, ratio)
  std::vector<int64_t> size(size_t(n) * R);
  std::vector<double> q(size_t(n) * MR), tt(size_t(n) * TT * MR), u(size_t(n) * TT * MR);
  std::vector<uint8_t> valid(size_t(n) * MR);
  if (n > 0 && (rc = kvt_score_candidates(h, p, tiers, n_tiers, space, params, size.data(), q.data(), valid.data(),
                                          tt.data(), u.data())))
    return rc;
  struct Cand {
    int t, m, r;
  };
  std::vector<std::vector<Cand>> cands(n);
  double assignments = 1.0;
  for (int c = 0; c < n; ++c) {
    auto& v = cands[c];
    for (int t = 0; t < TT; ++t)  // all_candidates order: tier, method, ratio (descending)
      for (int m = 0; m < M; ++m)
        for (int r = 0; r < R; ++r)
          if (valid[size_t(c) * MR + size_t(m) * R + r]) v.push_back({t, m, r});
    if (v.empty()) return set_error(KVT_EVALIDATION, "no scorable configuration for context " + std::to_string(c));
    auto U = [&](const Cand& x) { return u[(size_t(c) * TT + x.t) * MR + size_t(x.m) * R + x.r]; };
    auto Q = [&](const Cand& x) { return q[size_t(c) * MR + size_t(x.m) * R + x.r]; };
    std::stable_sort(v.begin(), v.end(), [&](const Cand& a, const Cand& b) {  // candidate_preferred (utility rule)
      if (U(a) != U(b)) return U(a) > U(b);
      if (Q(a) != Q(b)) return Q(a) > Q(b);
      if (T.id[a.t] != T.id[b.t]) return T.id[a.t] < T.id[b.t];
      if (S.ratio[a.r] != S.ratio[b.r]) return S.ratio[a.r] > S.ratio[b.r];
      return S.name_rank[a.m] < S.name_rank[b.m];
    });
    assignments *= static_cast<double>(v.size());
    if (assignments > max_assignments)
      return set_error(KVT_EVALIDATION, "instance too large for the exact solver: assignment space exceeds the limit");
  }
  // flattened candidates + the optimistic completion bound (right to left, like the reference)
  std::vector<double> cu_h;
  std::vector<long long> csz_h;
  std::vector<int> ct_h, off_h(n + 1, 0), cnt_h(n);
  for (int c = 0; c < n; ++c) {
    off_h[c] = static_cast<int>(cu_h.size());
    cnt_h[c] = static_cast<int>(cands[c].size());
    for (const Cand& x : cands[c]) {
      cu_h.push_back(u[(size_t(c) * TT + x.t) * MR + size_t(x.m) * R + x.r]);
      csz_h.push_back(size[size_t(c) * R + x.r]);
      ct_h.push_back(x.t);
    }
  }
  std::vector<double> suffix(n + 1, 0.0);
  for (int i = n; i-- > 0;) suffix[i] = suffix[i + 1] + cu_h[off_h[i]];
  // an incumbent for the shared prune: the first fitting candidate of every
  // context in order (a feasible total when it completes), lowered by a
  // relative 1e-12 so that rounding in the bounds never cuts the optimum
  double incumbent = -std::numeric_limits<double>::infinity();
  {
    std::vector<long long> used(TT, 0);
    double tot = 0.0;
    bool ok = true;
    for (int c = 0; c < n && ok; ++c) {
      ok = false;
      for (int k = 0; k < cnt_h[c]; ++k) {
        const int j = off_h[c] + k, t = ct_h[j];
        if (!T.unlimited[t] && used[t] + csz_h[j] > T.cap[t]) continue;
        used[t] += csz_h[j];
        tot += cu_h[j];
        ok = true;
        break;
      }
    }
    if (ok && n > 0) incumbent = tot - std::fabs(tot) * 1e-12 - 1e-300;
  }
  // subtrees: enough prefixes to fill the GPU when the space is large, few
  // when it is small (every thread's subtree is then tiny anyway)
  // subtrees (prefixes of the first d contexts) handed out dynamically to
  // persistent search threads: many more prefixes than threads when the
  // space is large (load balance), few when it is small
  const double space_sz = assignments;
  const long long nthreads = space_sz > 1e6 ? static_cast<long long>(num_sms_p() * 4) * 128 : 4096;
  const long long target = space_sz > 1e6 ? 64 * nthreads : 4096;
  int d = 0;
  long long nprefix = 1;
  while (d < n && nprefix * cnt_h[d] <= target) nprefix *= cnt_h[d++];
  // device buffers
  const size_t nc = std::max<size_t>(1, cu_h.size());
  const size_t bytes = nc * (8 + 8 + 4) + size_t(n + 1) * 4 * 2 + size_t(n + 1) * 8 + 16 +
                       size_t(nthreads) * (8 + 4 + 8 + 4 * size_t(std::max(n, 1))) + 64 * 10;
  char* dbuf = nullptr;
  KVT_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dbuf), bytes, h->stream));
  size_t o = 0;
  auto carve = [&](size_t b) {
    char* r = dbuf + o;
    o += (b + 63) & ~size_t(63);
    return r;
  };
  auto* d_cu = reinterpret_cast<double*>(carve(nc * 8));
  auto* d_csz = reinterpret_cast<long long*>(carve(nc * 8));
  auto* d_ct = reinterpret_cast<int*>(carve(nc * 4));
  auto* d_off = reinterpret_cast<int*>(carve(size_t(n + 1) * 4));
  auto* d_cnt = reinterpret_cast<int*>(carve(size_t(n + 1) * 4));
  auto* d_suf = reinterpret_cast<double*>(carve(size_t(n + 1) * 8));
  auto* d_gbest = reinterpret_cast<unsigned long long*>(carve(8));
  auto* d_next = reinterpret_cast<unsigned long long*>(carve(8));
  auto* d_tot = reinterpret_cast<double*>(carve(size_t(nthreads) * 8));
  auto* d_found = reinterpret_cast<int*>(carve(size_t(nthreads) * 4));
  auto* d_pfx = reinterpret_cast<long long*>(carve(size_t(nthreads) * 8));
  auto* d_choice = reinterpret_cast<int*>(carve(size_t(nthreads) * 4 * size_t(std::max(n, 1))));
  cudaStream_t st = h->stream;
  if (!cu_h.empty()) {
    KVT_CUDA_TRY(cudaMemcpyAsync(d_cu, cu_h.data(), cu_h.size() * 8, cudaMemcpyHostToDevice, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(d_csz, csz_h.data(), csz_h.size() * 8, cudaMemcpyHostToDevice, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(d_ct, ct_h.data(), ct_h.size() * 4, cudaMemcpyHostToDevice, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(d_off, off_h.data(), size_t(n) * 4, cudaMemcpyHostToDevice, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(d_cnt, cnt_h.data(), size_t(n) * 4, cudaMemcpyHostToDevice, st));
  }
  KVT_CUDA_TRY(cudaMemcpyAsync(d_suf, suffix.data(), size_t(n + 1) * 8, cudaMemcpyHostToDevice, st));
  {
    unsigned long long key = 0;  // key 0 < every real total's key (no incumbent)
    if (std::isfinite(incumbent)) {
      uint64_t b;
      std::memcpy(&b, &incumbent, 8);
      key = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
    }
    KVT_CUDA_TRY(cudaMemcpyAsync(d_gbest, &key, 8, cudaMemcpyHostToDevice, st));
    KVT_CUDA_TRY(cudaStreamSynchronize(st));  // key lives on this frame
  }
  KVT_CUDA_TRY(cudaMemsetAsync(d_next, 0, 8, st));
  auto kern = n <= kMckpSmallCtx ? k_mckp<kMckpSmallCtx> : k_mckp<kMckpMaxCtx>;
  kern<<<static_cast<int>((nthreads + 127) / 128), 128, 0, st>>>(d_cu, d_csz, d_ct, d_off, d_cnt, d_suf, T, n, d,
                                                                 nprefix, d_gbest, d_next, d_tot, d_found, d_pfx,
                                                                 d_choice);
  h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  auto* d_win = reinterpret_cast<long long*>(d_gbest);  // gbest is dead once the search is done
  k_mckp_pick<<<1, 1024, 0, st>>>(d_tot, d_found, d_pfx, nthreads, d_win);
  h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  long long win = -1;
  KVT_CUDA_TRY(cudaMemcpyAsync(&win, d_win, 8, cudaMemcpyDeviceToHost, st));
  KVT_CUDA_TRY(cudaStreamSynchronize(st));
  double best_total = 0.0;
  std::vector<int> choice_h(std::max(n, 1));
  if (win >= 0) {
    KVT_CUDA_TRY(cudaMemcpyAsync(&best_total, d_tot + win, 8, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(choice_h.data(), d_choice + size_t(win) * n, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
  }
  KVT_CUDA_TRY(cudaFreeAsync(dbuf, st));
  KVT_CUDA_TRY(cudaStreamSynchronize(st));
  if (win < 0) return set_error(KVT_EVALIDATION, "no feasible one-config-per-context assignment exists");
  *total_utility = best_total;
  for (int c = 0; c < n; ++c) {
    const Cand& x = cands[c][choice_h[c]];
    kvt_best& b = out[c];
    std::memset(&b, 0, sizeof b);
    b.tier_index = x.t;
    b.tier_id = T.id[x.t];
    b.method = x.m;
    b.ratio_index = x.r;
    b.ratio = S.ratio[x.r];
    b.size_bytes = size[size_t(c) * R + x.r];
    b.quality = q[size_t(c) * MR + size_t(x.m) * R + x.r];
    b.ttft = tt[(size_t(c) * TT + x.t) * MR + size_t(x.m) * R + x.r];
    b.utility = u[(size_t(c) * TT + x.t) * MR + size_t(x.m) * R + x.r];
  }
  return KVT_OK;
}

extern "C" int kvt_best_config(kvt_handle* h, const kvt_pset* p, const kvt_tier* tiers, int32_t n_tiers,
                               const kvt_space* space, const kvt_params* params, int32_t rule, kvt_best* out) {
  KVT_ON_DEVICE(h);
  DevSpace S;
  DevTiers T;
  int rc;
  if ((rc = resolve_space(space, &S))) return rc;
  if ((rc = resolve_tiers(tiers, n_tiers, &T))) return rc;
  if (p->dev.M != S.M) return set_error(KVT_EINVAL, "profile set / space method count mismatch");
  const size_t n = p->dev.n, R = S.R, MR = S.M * S.R, TMR = T.T * MR;
  const size_t b_size = n * R * 8, b_q = n * MR * 8, b_v = (n * MR + 255) & ~size_t(255), b_u = n * TMR * 8;
  const size_t b_best = n * sizeof(kvt_best);
  if ((rc = ensure_scratch(h, b_size + b_q + b_v + b_u + b_best + 1024))) return rc;
  char* b = static_cast<char*>(h->scratch);
  Tables t{reinterpret_cast<long long*>(b), reinterpret_cast<double*>(b + b_size),
           reinterpret_cast<unsigned char*>(b + b_size + b_q), nullptr,
           reinterpret_cast<double*>(b + b_size + b_q + b_v),
           reinterpret_cast<kvt_best*>(b + b_size + b_q + b_v + b_u)};
  if ((rc = launch_score(h, p->dev, S, T, params->alpha, rule, t))) return rc;
  KVT_CUDA_TRY(cudaMemcpyAsync(out, t.best, b_best, cudaMemcpyDeviceToHost, h->stream));
  KVT_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return KVT_OK;
}

// ------------------------------------------------------------------- store

enum : int {
  ST_OK = 0,
  ST_NEED_SPACE = 1,
  ST_ERR_RESIDENT = 2,     // already resident
  ST_ERR_NO_CONFIG = 3,    // best_config threw
  ST_ERR_NO_OPTION = 4,    // least_drop_update threw (no option)
  ST_ERR_QUALITY = 5,      // quality_of threw for a resident's current config
  ST_ERR_NOT_RESIDENT = 6,
  ST_ERR_TIER = 7,
};

struct Ctl {
  long long occ[KVT_MAX_TIERS];
  int errcount[KVT_MAX_TIERS];
  long long seq;
  long long n_act;
  long long cap_act;
  long long n_ops;
  long long resume_op;
  int in_resolve;
  int status;
  int err_ctx;
  int err_tier;
  int n_saved;
  int pad;
};

struct DevStore {
  int n;
  DevTiers TT;
  int* tier;       // tier index or -1
  int* meth;
  int* ridx;       // space ratio index or -1 (off grid)
  double* ratio;
  long long* orig;
  long long* freq;
  long long* last;
  long long* seq;
  // cached best update per resident (K2)
  double* cdrop;
  long long* cbytes;
  int* copt;       // enumeration index relative to the resident's tier; -1 none, -2 error
  int* mem;        // tree membership: tier index if in that tier's tree, else -1
  // 32-ary tournament trees, one per tier: tree[t*tree_stride + lvl_off[k] + node]
  // = winning resident (-1 none), tkey[same] = its (drop, bytes) key words
  int* tree;
  ulonglong2* tkey;
  int tree_stride;
  int nlev;
  int lvl_off[8];
  int lvl_size[8];
  kvt_action* act;
  Ctl* ctl;
  int* saved;      // rearrange order
};

struct StepCtx {
  DevStore st;
  DevProfiles P;
  DevSpace S;
  double alpha;
  Tables tb;
};

struct Key {
  double drop;
  long long bytes;
  int idx;
};

// update_preferred proj/src/placement.cpp:165-170 + enumeration order
__device__ __forceinline__ bool key_better(const Key& a, const Key& b) {
  if (a.idx < 0) return false;
  if (b.idx < 0) return true;
  if (a.drop != b.drop) return a.drop < b.drop;
  if (a.bytes != b.bytes) return a.bytes > b.bytes;
  return a.idx < b.idx;
}

// Keys as order-preserving unsigned words: a = drop (IEEE order, -0 folded
// into +0 like the reference's !=), b = bytes freed (larger first), c =
// index; the empty key (idx < 0) is all-ones and loses to any real key.
struct WKey {
  unsigned long long a, b;
  unsigned c;
};
__device__ __forceinline__ WKey wkey_empty() { return WKey{~0ull, ~0ull, ~0u}; }
__device__ __forceinline__ unsigned long long drop_word(double drop) {
  const unsigned long long d = static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(drop, 0.0)));
  return (d & 0x8000000000000000ull) ? ~d : (d | 0x8000000000000000ull);
}
__device__ __forceinline__ unsigned long long bytes_word(long long bytes) {
  return ~(static_cast<unsigned long long>(bytes) ^ 0x8000000000000000ull);
}
__device__ __forceinline__ WKey to_wkey(const Key& k) {
  if (k.idx < 0) return wkey_empty();
  return WKey{drop_word(k.drop), bytes_word(k.bytes), static_cast<unsigned>(k.idx)};
}
__device__ __forceinline__ Key from_wkey(const WKey& w) {
  Key r{0.0, 0, -1};
  if (w.c != ~0u) {
    const unsigned long long d = (w.a & 0x8000000000000000ull) ? (w.a & 0x7fffffffffffffffull) : ~w.a;
    r.drop = __longlong_as_double(static_cast<long long>(d));
    r.bytes = static_cast<long long>(~w.b ^ 0x8000000000000000ull);
    r.idx = static_cast<int>(w.c);
  }
  return r;
}

// Warp argmin under key_better's total order: five 32-bit warp min
// reductions (REDUX) over the key words, each narrowing the candidate lanes.
__device__ __forceinline__ WKey warp_min_w(const WKey& k) {
  const unsigned lane_bit = 1u << (threadIdx.x & 31);
  unsigned cand = 0xffffffffu;
  auto step = [&](unsigned x) {
    const unsigned m = __reduce_min_sync(0xffffffffu, (cand & lane_bit) ? x : ~0u);
    cand &= __ballot_sync(0xffffffffu, x == m);
    return m;
  };
  step(static_cast<unsigned>(k.a >> 32));
  if (__popc(cand) != 1) {  // ties on the high drop word (or no key at all): narrow on the rest
    step(static_cast<unsigned>(k.a));
    step(static_cast<unsigned>(k.b >> 32));
    step(static_cast<unsigned>(k.b));
    step(k.c);
  }
  const int src = __ffs(cand) - 1;  // the winner (lowest lane among equal keys: all words equal)
  return WKey{__shfl_sync(0xffffffffu, k.a, src), __shfl_sync(0xffffffffu, k.b, src), __shfl_sync(0xffffffffu, k.c, src)};
}
__device__ __forceinline__ Key warp_min(const Key& k) { return from_wkey(warp_min_w(to_wkey(k))); }

// score_candidate proj/src/utility.cpp:65-79 for an arbitrary ratio.
__device__ __forceinline__ bool score_fly(const StepCtx& X, int c, int t, int m, double ratio, double* u,
                                          long long* size, double* q_out = nullptr, double* tt_out = nullptr) {
  double q;
  if (!quality_of(X.P, c, m, ratio, &q)) return false;
  const long long sz = csize(X.P.orig[c], ratio);
  const double tt = load_time(sz, X.st.TT.lat[t], X.st.TT.bw[t], X.S.ovh[m]);
  *u = utility_score(q, tt, X.P.freq[c], X.alpha);
  *size = sz;
  if (q_out) *q_out = q;
  if (tt_out) *tt_out = tt;
  return true;
}

// K2: best update of one resident (enumerate_updates proj/src/utility.cpp:
// 81-127 scored against its current candidate, placement.cpp:179-197).
// Whole warp; lane 0 writes the cache. Returns the best key (idx = the
// option's enumeration index, -1 none); *member = the tree membership.
// Every table load of a step is issued before any of them is consumed.
__device__ Key compute_cache(const StepCtx& X, int c, int cur, int me, int re, double rate, long long eorig,
                             int* member = nullptr) {
  const int lane = threadIdx.x & 31;
  const int M = X.S.M, R = X.S.R, T = X.st.TT.T, MR = M * R;
  const size_t qb = static_cast<size_t>(c) * MR;
  const int per = MR + 1, nj = T - cur;
  // the (method, ratio) grid in every tier >= cur, option w = lane + 32 q:
  // its table loads go out first, with the current config's
  constexpr int kQ = 3, kJ = 4;
  bool gv[kQ];
  long long gso[kQ];
  double gratio[kQ], guo[kQ][kJ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    const int w = lane + 32 * q;
    gv[q] = false;
    if (w < MR) {
      const int r = w % R;
      gv[q] = X.tb.valid[qb + w] != 0;
      gso[q] = X.tb.size[static_cast<size_t>(c) * R + r];
      gratio[q] = X.S.ratio[r];
#pragma unroll
      for (int j = 0; j < kJ; ++j)
        if (j < nj) guo[q][j] = X.tb.u[(static_cast<size_t>(c) * T + cur + j) * MR + w];
    }
  }
  const int rr = re >= 0 ? re : 0;
  const bool cov_v = X.tb.valid[qb + static_cast<size_t>(me) * R + rr] != 0;
  const double ucov = X.tb.u[(static_cast<size_t>(c) * T + cur) * MR + static_cast<size_t>(me) * R + rr];
  const long long scov = X.tb.size[static_cast<size_t>(c) * R + rr];
  const bool covered = re >= 0 && cov_v;
  double ucur = ucov;
  long long scur = scov;
  bool ok = true;
  if (!covered) ok = score_fly(X, c, cur, me, rate, &ucur, &scur);
  if (!ok) {
    if (lane == 0) {
      X.st.copt[c] = -2;
      X.st.mem[c] = -1;
      atomicAdd(&X.st.ctl->errcount[cur], 1);
    }
    __syncwarp();
    if (member) *member = -1;
    return Key{0.0, 0, -1};
  }
  const long long cur_bytes = csize(eorig, rate);
  Key best{0.0, 0, -1};
  auto consider = [&](const Key& k) {
    if (key_better(k, best)) best = k;
  };
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    const int w = lane + 32 * q;
    if (w < MR && gv[q]) {
      const bool shrinks = csize(eorig, gratio[q]) < cur_bytes;
#pragma unroll
      for (int j = 0; j < kJ; ++j)
        if (j < nj && (j > 0 || shrinks)) consider(Key{__dsub_rn(ucur, guo[q][j]), j == 0 ? scur - gso[q] : scur, j * per + w});
      for (int j = kJ; j < nj; ++j)  // more than kJ tiers below
        consider(Key{__dsub_rn(ucur, X.tb.u[(static_cast<size_t>(c) * T + cur + j) * MR + w]), scur, j * per + w});
    }
  }
  for (int w = lane + 32 * kQ; w < MR; w += 32) {  // larger spaces
    if (X.tb.valid[qb + w] == 0) continue;
    const int r = w % R;
    const long long so = X.tb.size[static_cast<size_t>(c) * R + r];
    const bool shrinks = csize(eorig, X.S.ratio[r]) < cur_bytes;
    for (int j = 0; j < nj; ++j)
      if (j > 0 || shrinks)
        consider(Key{__dsub_rn(ucur, X.tb.u[(static_cast<size_t>(c) * T + cur + j) * MR + w]), j == 0 ? scur - so : scur,
                     j * per + w});
  }
  // keep an off-grid config and move it down a tier (option w = MR)
  if (lane == MR % 32 && !covered && scorable(X.P, c, me, rate)) {
    for (int j = 1; j < nj; ++j) {
      double uo;
      long long so;
      if (score_fly(X, c, cur + j, me, rate, &uo, &so)) consider(Key{__dsub_rn(ucur, uo), scur, j * per + MR});
    }
  }
  best = warp_min(best);
  const int mem = best.idx >= 0 ? cur : -1;
  if (lane == 0) {
    X.st.cdrop[c] = best.drop;
    X.st.cbytes[c] = best.bytes;
    X.st.copt[c] = best.idx;
    X.st.mem[c] = mem;
  }
  __syncwarp();
  if (member) *member = mem;
  return best;
}

__device__ __forceinline__ Key leaf_key(const DevStore& st, int i, int t) {
  Key k{0.0, 0, -1};
  if (i < st.n && st.mem[i] == t) {
    k.drop = st.cdrop[i];
    k.bytes = st.cbytes[i];
    k.idx = i;
  }
  return k;
}
// leaf i of tier t's tree; the three loads are issued unconditionally
__device__ __forceinline__ WKey leaf_wkey(const DevStore& st, int i, int t) {
  if (i >= st.n) return wkey_empty();
  const int mem = st.mem[i];
  const double d = st.cdrop[i];
  const long long b = st.cbytes[i];
  return mem == t ? WKey{drop_word(d), bytes_word(b), static_cast<unsigned>(i)} : wkey_empty();
}
__device__ __forceinline__ size_t node_at(const DevStore& st, int t, int l, int node) {
  return static_cast<size_t>(t) * st.tree_stride + st.lvl_off[l] + node;
}
__device__ __forceinline__ WKey node_wkey(const DevStore& st, int t, int l, int node) {
  const size_t at = node_at(st, t, l, node);
  const ulonglong2 ab = st.tkey[at];
  return WKey{ab.x, ab.y, static_cast<unsigned>(st.tree[at])};
}
__device__ __forceinline__ void node_store(const DevStore& st, int t, int l, int node, const WKey& k) {
  const size_t at = node_at(st, t, l, node);
  st.tree[at] = static_cast<int>(k.c);
  st.tkey[at] = make_ulonglong2(k.a, k.b);
}

// A leaf-to-root path of one tier's tree: the 31 siblings of every path
// node, loaded in one round (they do not depend on the new leaf key).
constexpr int kMaxLev = 6;  // 32^6 residents
struct TreePath {
  WKey sib[kMaxLev];
};
__device__ __forceinline__ void path_load(const DevStore& st, int t, int c, TreePath& p) {
  const int lane = threadIdx.x & 31;
  int node = c >> 5;
  p.sib[0] = leaf_wkey(st, (node << 5) + lane, t);
#pragma unroll
  for (int l = 1; l < kMaxLev; ++l) {
    if (l < st.nlev) {
      node >>= 5;
      const int i = (node << 5) + lane;
      p.sib[l] = i < st.lvl_size[l - 1] ? node_wkey(st, t, l - 1, i) : wkey_empty();
    }
  }
}
// Recompute the path with leaf c's new key (whole warp); returns the root.
__device__ __forceinline__ WKey path_finish(const DevStore& st, int t, int c, const TreePath& p, WKey k) {
  const int lane = threadIdx.x & 31;
  int child = c;
#pragma unroll
  for (int l = 0; l < kMaxLev; ++l) {
    if (l < st.nlev) {
      k = warp_min_w(lane == (child & 31) ? k : p.sib[l]);
      child >>= 5;
      if (lane == 0) node_store(st, t, l, child, k);
    }
  }
  __syncwarp();
  return k;
}
// leaf c's key in tier t's tree after compute_cache (member = its tree)
__device__ __forceinline__ WKey member_wkey(const Key& best, int member, int t, int c) {
  return member == t && best.idx >= 0 ? WKey{drop_word(best.drop), bytes_word(best.bytes), static_cast<unsigned>(c)}
                                      : wkey_empty();
}

__device__ __forceinline__ int tree_root(const DevStore& st, int t) {
  return st.tree[node_at(st, t, st.nlev - 1, 0)];
}

struct Ops {
  const int* ctx;
  const long long* freq;  // null: use the store's saved stats (rearrange)
  const long long* stamp;
};

// K3: persistent single-warp greedy. Processes ops[resume_op..n_ops):
// insert_joint (placement.cpp:225-250) then resolve_overflow (206-223).
__global__ void __launch_bounds__(32, 1) k_greedy(StepCtx X, Ops ops) {
  const int lane = threadIdx.x;
  DevStore& st = X.st;
  Ctl* ctl = st.ctl;
  const int T = st.TT.T, MR = X.S.M * X.S.R, R = X.S.R;
  long long occ = lane < T ? ctl->occ[lane] : 0;
  const long long capv = lane < T ? st.TT.cap[lane] : 0;
  const bool finite = lane < T && !st.TT.unlimited[lane];
  long long op = ctl->resume_op;
  bool in_resolve = ctl->in_resolve != 0;
  long long nact = ctl->n_act, seq = ctl->seq;
  const long long cap_act = ctl->cap_act, n_ops = ctl->n_ops;
  int status = ST_OK, err_ctx = -1, err_tier = -1;
  // lane t keeps tier t's tree root; this warp is the trees' only writer
  unsigned root = lane < T && finite ? static_cast<unsigned>(tree_root(st, lane)) : ~0u;

  while (true) {
    if (!in_resolve) {
      if (op >= n_ops) break;
      const int c = ops.ctx[op];
      if (st.tier[c] >= 0) {
        status = ST_ERR_RESIDENT;
        err_ctx = c;
        break;
      }
      const kvt_best b = X.tb.best[c];
      if (b.status != 0) {
        status = ST_ERR_NO_CONFIG;
        err_ctx = c;
        break;
      }
      if (nact >= cap_act) {
        status = ST_NEED_SPACE;
        break;
      }
      const long long eorig = X.P.orig[c];
      const long long sz = csize(eorig, b.ratio);
      if (lane == b.tier_index) occ += sz;
      if (lane == 0) {
        st.tier[c] = b.tier_index;
        st.meth[c] = b.method;
        st.ridx[c] = b.ratio_index;
        st.ratio[c] = b.ratio;
        st.orig[c] = eorig;
        st.freq[c] = ops.freq ? ops.freq[op] : st.freq[c];
        st.last[c] = ops.freq ? ops.stamp[op] : st.last[c];
        st.seq[c] = seq;
        kvt_action a;
        a.kind = KVT_INSERT;
        a.ctx = c;
        a.tier_id = b.tier_id;
        a.method = b.method;
        a.ratio = b.ratio;
        st.act[nact] = a;
      }
      ++seq;
      ++nact;
      __syncwarp();
      const bool fin = !st.TT.unlimited[b.tier_index];
      TreePath path;
      if (fin) path_load(st, b.tier_index, c, path);
      int member;
      const Key k = compute_cache(X, c, b.tier_index, b.method, b.ratio_index, b.ratio, eorig, &member);
      if (fin) {
        const WKey r = path_finish(st, b.tier_index, c, path, member_wkey(k, member, b.tier_index, c));
        if (lane == b.tier_index) root = r.c;
      }
      in_resolve = true;
    }
    // resolve_overflow: topmost over-full finite tier first (placement.cpp:54-59,211)
    const unsigned over = __ballot_sync(0xffffffffu, finite && occ > capv);
    if (over == 0) {
      in_resolve = false;
      ++op;
      continue;
    }
    const int t = __ffs(over) - 1;
    if (nact >= cap_act) {
      status = ST_NEED_SPACE;
      break;
    }
    if (ctl->errcount[t] > 0) {
      status = ST_ERR_QUALITY;
      err_tier = t;
      break;
    }
    const int w = static_cast<int>(__shfl_sync(0xffffffffu, root, t));
    if (w < 0) {
      status = ST_ERR_NO_OPTION;
      err_tier = t;
      break;
    }
    // apply the winner's cached option (placement.cpp:213-221)
    const int e = st.copt[w];
    const int me = st.meth[w], re = st.ridx[w];
    const double rate = st.ratio[w];
    const long long eorig = st.orig[w];
    const int per = MR + 1;
    const int j = e / per, wi = e - j * per, ti = t + j;
    int nm, nr;
    double nratio;
    if (wi < MR) {
      nm = wi / R;
      nr = wi - nm * R;
      nratio = X.S.ratio[nr];
    } else {
      nm = me;
      nr = re;
      nratio = rate;
    }
    const long long oldb = csize(eorig, rate), newb = csize(eorig, nratio);
    if (ti == t) {
      if (lane == t) occ += newb - oldb;
    } else {
      if (lane == t) occ -= oldb;
      if (lane == ti) occ += newb;
    }
    if (lane == 0) {
      st.meth[w] = nm;
      st.ridx[w] = nr;
      st.ratio[w] = nratio;
      if (ti != t) {
        st.tier[w] = ti;
        st.seq[w] = seq;
      }
      kvt_action a;
      a.kind = ti == t ? KVT_RECOMPRESS : KVT_EVICT;
      a.ctx = w;
      a.tier_id = st.TT.id[ti];
      a.method = nm;
      a.ratio = nratio;
      st.act[nact] = a;
    }
    if (ti != t) ++seq;
    ++nact;
    __syncwarp();
    const bool fin2 = ti != t && !st.TT.unlimited[ti];
    TreePath p1, p2;
    path_load(st, t, w, p1);
    if (fin2) path_load(st, ti, w, p2);
    int member;
    const Key k = compute_cache(X, w, ti, nm, nr, nratio, eorig, &member);
    const WKey r1 = path_finish(st, t, w, p1, member_wkey(k, member, t, w));
    if (lane == t) root = r1.c;
    if (fin2) {
      const WKey r2 = path_finish(st, ti, w, p2, member_wkey(k, member, ti, w));
      if (lane == ti) root = r2.c;
    }
  }
  if (lane < T) ctl->occ[lane] = occ;
  if (lane == 0) {
    ctl->resume_op = op;
    ctl->in_resolve = in_resolve ? 1 : 0;
    ctl->n_act = nact;
    ctl->seq = seq;
    ctl->status = status;
    ctl->err_ctx = err_ctx;
    ctl->err_tier = err_tier;
  }
}

// Rebuild every resident's cache (warp per context) after profile/space
// changes or direct StoreState edits.
__global__ void __launch_bounds__(128) k_rebuild_cache(StepCtx X) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= X.st.n) return;
  const int t = X.st.tier[c];
  if (t < 0) {
    if ((threadIdx.x & 31) == 0) {
      X.st.mem[c] = -1;
      X.st.copt[c] = -1;
    }
    return;
  }
  // re-resolve the on-grid ratio index against the current space (exact ==,
  // CompressionConfig::operator==, proj/include/kvtier/core.hpp:55-57)
  const double rate = X.st.ratio[c];
  int re = -1;
  for (int r = 0; r < X.S.R; ++r)
    if (X.S.ratio[r] == rate) re = r;
  if ((threadIdx.x & 31) == 0) X.st.ridx[c] = re;
  compute_cache(X, c, t, X.st.meth[c], re, rate, X.st.orig[c]);
}

// Build one tree level for every tier (warp per node).
__global__ void __launch_bounds__(128) k_tree_level(DevStore st, int lvl, int t0) {
  const int node = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int t = t0 + blockIdx.y;
  if (node >= st.lvl_size[lvl]) return;
  const int i = (node << 5) + lane;
  WKey k = wkey_empty();
  if (lvl == 0) k = leaf_wkey(st, i, t);
  else if (i < st.lvl_size[lvl - 1]) k = node_wkey(st, t, lvl - 1, i);
  k = warp_min_w(k);
  if (lane == 0) node_store(st, t, lvl, node, k);
}

// Direct StoreState edits (placement.cpp:91-142); one thread.
enum { OP_ADD, OP_REMOVE, OP_RECONF, OP_TOUCH };
__global__ void k_store_op(DevStore st, int op, int c, kvt_entry e, kvt_entry* removed) {
  Ctl* ctl = st.ctl;
  ctl->status = ST_OK;
  ctl->err_ctx = c;
  const int t = st.tier[c];
  if (op == OP_ADD) {
    if (t >= 0) {
      ctl->status = ST_ERR_RESIDENT;
      return;
    }
    st.tier[c] = e.tier_index;
    st.meth[c] = e.method;
    st.ridx[c] = e.seq;  // host passes the resolved ratio index in seq
    st.ratio[c] = e.ratio;
    st.orig[c] = e.original_size_bytes;
    st.freq[c] = e.frequency;
    st.last[c] = e.last_access;
    st.seq[c] = ctl->seq++;
    ctl->occ[e.tier_index] += csize(e.original_size_bytes, e.ratio);
    return;
  }
  if (t < 0) {
    ctl->status = ST_ERR_NOT_RESIDENT;
    return;
  }
  if (op == OP_REMOVE) {
    removed->tier_index = t;
    removed->method = st.meth[c];
    removed->ratio = st.ratio[c];
    removed->original_size_bytes = st.orig[c];
    removed->frequency = st.freq[c];
    removed->last_access = st.last[c];
    removed->seq = st.seq[c];
    ctl->occ[t] -= csize(st.orig[c], st.ratio[c]);
    st.tier[c] = -1;
    st.mem[c] = -1;
  } else if (op == OP_RECONF) {
    ctl->occ[t] += csize(st.orig[c], e.ratio) - csize(st.orig[c], st.ratio[c]);
    st.meth[c] = e.method;
    st.ratio[c] = e.ratio;
    st.ridx[c] = e.seq;
  } else {
    st.freq[c] += 1;
    st.last[c] = e.last_access;
  }
}

// least_drop_update query: the root of tier t with its option spelled out.
__global__ void k_ld_query(StepCtx X, int t, kvt_update* out) {
  const DevStore& st = X.st;
  Ctl* ctl = st.ctl;
  ctl->status = ST_OK;
  if (ctl->errcount[t] > 0) {
    ctl->status = ST_ERR_QUALITY;
    ctl->err_tier = t;
    return;
  }
  const int w = tree_root(st, t);
  if (w < 0) {
    ctl->status = ST_ERR_NO_OPTION;
    ctl->err_tier = t;
    return;
  }
  const int MR = X.S.M * X.S.R, R = X.S.R;
  const int e = st.copt[w], per = MR + 1, j = e / per, wi = e - j * per, ti = t + j;
  int nm;
  double nratio;
  if (wi < MR) {
    nm = wi / R;
    nratio = X.S.ratio[wi - nm * R];
  } else {
    nm = st.meth[w];
    nratio = st.ratio[w];
  }
  kvt_update u = {};
  u.ctx = w;
  u.kind = ti == t ? KVT_RECOMPRESS : KVT_EVICT;
  u.tier_index = ti;
  u.tier_id = st.TT.id[ti];
  u.method = nm;
  u.ratio = nratio;
  long long sz = 0;
  score_fly(X, w, ti, nm, nratio, &u.utility, &sz, &u.quality, &u.ttft);
  u.size_bytes = sz;
  u.utility_drop = st.cdrop[w];
  u.bytes_freed = st.cbytes[w];
  *out = u;
}

// rearrange (placement.cpp:252-283) sort keys: utility descending, then
// context ascending (stable radix sort over contexts in index order).
__global__ void k_rearrange_keys(DevStore st, const kvt_best* best, unsigned long long* keys, int* vals) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= st.n) return;
  vals[c] = c;
  if (st.tier[c] < 0) {
    keys[c] = ~0ull;
    return;
  }
  if (best[c].status != 0) {
    st.ctl->status = ST_ERR_NO_CONFIG;
    st.ctl->err_ctx = c;
  }
  double u = best[c].utility;
  if (u == 0.0) u = 0.0;  // -0.0 == +0.0 in the reference's comparator
  unsigned long long b = __double_as_longlong(u);
  b = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);  // ascending order key
  keys[c] = ~b;  // descending utility
  atomicAdd(&st.ctl->n_saved, 1);
}

__global__ void k_clear(DevStore st) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < st.n) {
    st.tier[c] = -1;
    st.mem[c] = -1;
    st.copt[c] = -1;
  }
  if (c < KVT_MAX_TIERS) {
    st.ctl->occ[c] = 0;
    st.ctl->errcount[c] = 0;
  }
}

// placement_utility (placement.cpp:285-298): per-resident utility, then an
// ordered (tier, arrival) sum by one thread so the FP sum order matches.
__global__ void k_util_terms(StepCtx X, double* term, unsigned long long* keys, int* vals, int* bad) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= X.st.n) return;
  vals[c] = c;
  const int t = X.st.tier[c];
  if (t < 0) {
    keys[c] = ~0ull;
    term[c] = 0.0;
    return;
  }
  // occupancy-side size uses the entry's size (CacheEntry::compressed_bytes)
  double q;
  if (!quality_of(X.P, c, X.st.meth[c], X.st.ratio[c], &q)) {
    *bad = c + 1;
    term[c] = 0.0;
  } else {
    const long long sz = csize(X.st.orig[c], X.st.ratio[c]);
    const double tt = load_time(sz, X.st.TT.lat[t], X.st.TT.bw[t], X.S.ovh[X.st.meth[c]]);
    term[c] = utility_score(q, tt, X.P.freq[c], X.alpha);
  }
  keys[c] = (static_cast<unsigned long long>(t) << 56) | static_cast<unsigned long long>(X.st.seq[c]);
}

__global__ void k_util_sum(const double* term, const int* order, int n_res, double* out) {
  double total = 0.0;
  for (int i = 0; i < n_res; ++i) total = __dadd_rn(total, term[order[i]]);
  *out = total;
}

struct kvt_store {
  kvt_handle* h = nullptr;
  DevStore d{};
  DevTiers TT{};
  int n = 0;
  void* buf = nullptr;
  // tables for this store's tiers
  void* tbuf = nullptr;
  size_t tbytes = 0;
  Tables tb{};
  uint64_t tkey = 0;
  bool cache_dirty = true;
  uint64_t cache_key = 0;
  long long cap_act = 0;
  kvt_action* act = nullptr;
  int* ops_buf = nullptr;
  long long* ops_l = nullptr;
  long long ops_cap = 0;
  std::vector<std::string> names;
  bool has_space = false;
  DevSpace S{};
};

static int store_fetch_ctl(kvt_store* s, Ctl* c) {
  KVT_CUDA_TRY(cudaMemcpyAsync(c, s->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s->h->stream));
  KVT_CUDA_TRY(cudaStreamSynchronize(s->h->stream));
  return KVT_OK;
}

extern "C" int kvt_store_create(kvt_handle* h, const kvt_tier* tiers, int32_t n_tiers, int32_t n_ctx,
                                kvt_store** out) {
  KVT_ON_DEVICE(h);
  DevTiers T;
  int rc;
  if ((rc = resolve_tiers(tiers, n_tiers, &T))) return rc;
  if (n_ctx < 0) return set_error(KVT_EINVAL, "negative context count");
  auto* s = new kvt_store();
  s->h = h;
  s->TT = T;
  s->n = n_ctx;
  DevStore& d = s->d;
  d.n = n_ctx;
  d.TT = T;
  // tree levels
  int sz = std::max(1, (n_ctx + 31) / 32), nl = 0, off = 0;
  while (true) {
    d.lvl_off[nl] = off;
    d.lvl_size[nl] = sz;
    off += sz;
    ++nl;
    if (sz == 1) break;
    sz = (sz + 31) / 32;
  }
  d.nlev = nl;
  d.tree_stride = off;
  const size_t n = std::max(1, n_ctx);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t o = 0;
  auto carve = [&](size_t bytes) {
    size_t at = o;
    o += align(bytes);
    return at;
  };
  const size_t o_tier = carve(4 * n), o_meth = carve(4 * n), o_ridx = carve(4 * n), o_ratio = carve(8 * n),
               o_orig = carve(8 * n), o_freq = carve(8 * n), o_last = carve(8 * n), o_seq = carve(8 * n),
               o_cdrop = carve(8 * n), o_cbytes = carve(8 * n), o_copt = carve(4 * n), o_mem = carve(4 * n),
               o_tree = carve(4 * static_cast<size_t>(off) * T.T),
               o_tkey = carve(sizeof(ulonglong2) * static_cast<size_t>(off) * T.T), o_ctl = carve(sizeof(Ctl)),
               o_saved = carve(4 * n);
  cudaError_t e = cudaMalloc(&s->buf, o);
  if (e != cudaSuccess) {
    delete s;
    return set_error(KVT_ECUDA, std::string("cudaMalloc store: ") + cudaGetErrorString(e));
  }
  char* b = static_cast<char*>(s->buf);
  d.tier = reinterpret_cast<int*>(b + o_tier);
  d.meth = reinterpret_cast<int*>(b + o_meth);
  d.ridx = reinterpret_cast<int*>(b + o_ridx);
  d.ratio = reinterpret_cast<double*>(b + o_ratio);
  d.orig = reinterpret_cast<long long*>(b + o_orig);
  d.freq = reinterpret_cast<long long*>(b + o_freq);
  d.last = reinterpret_cast<long long*>(b + o_last);
  d.seq = reinterpret_cast<long long*>(b + o_seq);
  d.cdrop = reinterpret_cast<double*>(b + o_cdrop);
  d.cbytes = reinterpret_cast<long long*>(b + o_cbytes);
  d.copt = reinterpret_cast<int*>(b + o_copt);
  d.mem = reinterpret_cast<int*>(b + o_mem);
  d.tree = reinterpret_cast<int*>(b + o_tree);
  d.tkey = reinterpret_cast<ulonglong2*>(b + o_tkey);
  d.ctl = reinterpret_cast<Ctl*>(b + o_ctl);
  d.saved = reinterpret_cast<int*>(b + o_saved);
  cudaStream_t st = h->stream;
  cudaMemsetAsync(s->buf, 0, o, st);
  cudaMemsetAsync(d.tier, 0xff, 4 * n, st);
  cudaMemsetAsync(d.mem, 0xff, 4 * n, st);
  cudaMemsetAsync(d.copt, 0xff, 4 * n, st);
  cudaMemsetAsync(d.tree, 0xff, 4 * static_cast<size_t>(off) * T.T, st);
  cudaMemsetAsync(d.tkey, 0xff, sizeof(ulonglong2) * static_cast<size_t>(off) * T.T, st);
  s->cap_act = 4096;
  e = cudaMalloc(&s->act, sizeof(kvt_action) * s->cap_act);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cudaFree(s->buf);
    delete s;
    return set_error(KVT_ECUDA, std::string("store init: ") + cudaGetErrorString(e));
  }
  d.act = s->act;
  *out = s;
  return KVT_OK;
}

extern "C" int kvt_store_destroy(kvt_store* s) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  if (!s) return KVT_OK;
  cudaFree(s->buf);
  cudaFree(s->tbuf);
  cudaFree(s->act);
  cudaFree(s->ops_buf);
  cudaFree(s->ops_l);
  delete s;
  return KVT_OK;
}

extern "C" int kvt_store_bind_space(kvt_store* s, const kvt_space* space) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  DevSpace S;
  int rc;
  if ((rc = resolve_space(space, &S))) return rc;
  s->S = S;
  s->has_space = true;
  return KVT_OK;
}

static int ratio_index(const kvt_store* s, double ratio) {
  if (!s->has_space) return -1;
  for (int r = 0; r < s->S.R; ++r)
    if (s->S.ratio[r] == ratio) return r;
  return -1;
}

static int store_status_error(kvt_store* s, const Ctl& c) {
  const std::string ctx = std::to_string(c.err_ctx);
  switch (c.status) {
    case ST_OK:
      return KVT_OK;
    case ST_ERR_RESIDENT:
      return set_error(KVT_EVALIDATION, "context " + ctx + " is already resident");
    case ST_ERR_NO_CONFIG:
      return set_error(KVT_EVALIDATION, "no scorable configuration for context " + ctx);
    case ST_ERR_NO_OPTION:
      return set_error(KVT_EVALIDATION, "tier " + std::to_string(s->TT.id[c.err_tier]) +
                                            " is over capacity and no resident has a space-saving option");
    case ST_ERR_QUALITY:
      return set_error(KVT_EVALIDATION, "a resident of tier " + std::to_string(s->TT.id[c.err_tier]) +
                                            " has a configuration its profile cannot score");
    case ST_ERR_NOT_RESIDENT:
      return set_error(KVT_EVALIDATION, "context " + ctx + " is not resident");
    default:
      return set_error(KVT_EINVAL, "store kernel status " + std::to_string(c.status));
  }
}

static int run_store_op(kvt_store* s, int op, int c, const kvt_entry& e, kvt_entry* removed) {
  if (c < 0 || c >= s->n) return set_error(KVT_EINVAL, "context index out of range");
  kvt_entry* d_removed = nullptr;
  if (removed) KVT_CUDA_TRY(cudaMallocAsync(&d_removed, sizeof(kvt_entry), s->h->stream));
  k_store_op<<<1, 1, 0, s->h->stream>>>(s->d, op, c, e, d_removed);
  s->h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  if (removed) {
    KVT_CUDA_TRY(cudaMemcpyAsync(removed, d_removed, sizeof(kvt_entry), cudaMemcpyDeviceToHost, s->h->stream));
    KVT_CUDA_TRY(cudaFreeAsync(d_removed, s->h->stream));
  }
  Ctl c2;
  int rc = store_fetch_ctl(s, &c2);
  if (rc) return rc;
  if (op != OP_TOUCH) s->cache_dirty = true;
  return store_status_error(s, c2);
}

extern "C" int kvt_store_add(kvt_store* s, int32_t ctx, const kvt_entry* e) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  if (e->tier_index < 0 || e->tier_index >= s->TT.T)
    return set_error(KVT_EVALIDATION, "unknown tier index " + std::to_string(e->tier_index));
  if (e->original_size_bytes <= 0) return set_error(KVT_EVALIDATION, "original size must be > 0");
  if (!(e->ratio > 0.0) || e->ratio > 1.0 || !std::isfinite(e->ratio))
    return set_error(KVT_EVALIDATION, "compression ratio must be in (0, 1]");
  if (s->has_space && (e->method < 0 || e->method >= s->S.M))
    return set_error(KVT_EVALIDATION, "unknown compression method index");
  kvt_entry x = *e;
  x.seq = ratio_index(s, e->ratio);
  return run_store_op(s, OP_ADD, ctx, x, nullptr);
}

extern "C" int kvt_store_remove(kvt_store* s, int32_t ctx, kvt_entry* removed) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  kvt_entry x{};
  kvt_entry tmp{};
  return run_store_op(s, OP_REMOVE, ctx, x, removed ? removed : &tmp);
}

extern "C" int kvt_store_reconfigure(kvt_store* s, int32_t ctx, int32_t m, double ratio) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  if (!(ratio > 0.0) || ratio > 1.0 || !std::isfinite(ratio))
    return set_error(KVT_EVALIDATION, "compression ratio must be in (0, 1]");
  kvt_entry x{};
  x.method = m;
  x.ratio = ratio;
  x.seq = ratio_index(s, ratio);
  return run_store_op(s, OP_RECONF, ctx, x, nullptr);
}

// n StoreState::touch calls in order, one thread (a later touch of the same
// context must win last_access); stops at the first non-resident context.
__global__ void k_touch_many(DevStore st, const int32_t* ctx, const int64_t* stamps, int64_t n) {
  Ctl* ctl = st.ctl;
  ctl->status = ST_OK;
  for (int64_t i = 0; i < n; ++i) {
    const int c = ctx[i];
    if (c < 0 || c >= st.n || st.tier[c] < 0) {
      ctl->status = ST_ERR_NOT_RESIDENT;
      ctl->err_ctx = c;
      return;
    }
    st.freq[c] += 1;
    st.last[c] = stamps[i];
  }
}

extern "C" int kvt_store_touch_many(kvt_store* s, const int32_t* ctx, const int64_t* stamps, int64_t n) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  if (n <= 0) return KVT_OK;
  char* d = nullptr;
  const size_t bc = sizeof(int32_t) * size_t(n), bs = sizeof(int64_t) * size_t(n);
  KVT_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), bs + bc, s->h->stream));
  KVT_CUDA_TRY(cudaMemcpyAsync(d, stamps, bs, cudaMemcpyHostToDevice, s->h->stream));
  KVT_CUDA_TRY(cudaMemcpyAsync(d + bs, ctx, bc, cudaMemcpyHostToDevice, s->h->stream));
  k_touch_many<<<1, 1, 0, s->h->stream>>>(s->d, reinterpret_cast<const int32_t*>(d + bs),
                                          reinterpret_cast<const int64_t*>(d), n);
  s->h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  KVT_CUDA_TRY(cudaFreeAsync(d, s->h->stream));
  Ctl c2;
  int rc = store_fetch_ctl(s, &c2);
  if (rc) return rc;
  return store_status_error(s, c2);
}

extern "C" int kvt_store_touch(kvt_store* s, int32_t ctx, int64_t stamp) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  kvt_entry x{};
  x.last_access = stamp;
  return run_store_op(s, OP_TOUCH, ctx, x, nullptr);
}

extern "C" int kvt_store_clear(kvt_store* s) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  k_clear<<<(s->n + 255) / 256 + 1, 256, 0, s->h->stream>>>(s->d);
  s->h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  KVT_CUDA_TRY(cudaMemsetAsync(s->d.tree, 0xff, 4 * static_cast<size_t>(s->d.tree_stride) * s->TT.T, s->h->stream));
  KVT_CUDA_TRY(cudaMemsetAsync(s->d.tkey, 0xff, sizeof(ulonglong2) * static_cast<size_t>(s->d.tree_stride) * s->TT.T,
                               s->h->stream));
  KVT_CUDA_TRY(cudaStreamSynchronize(s->h->stream));
  return KVT_OK;
}

extern "C" int kvt_store_occupancy(kvt_store* s, int64_t* occ) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  Ctl c;
  int rc = store_fetch_ctl(s, &c);
  if (rc) return rc;
  for (int t = 0; t < s->TT.T; ++t) occ[t] = c.occ[t];
  return KVT_OK;
}

extern "C" int kvt_store_snapshot(kvt_store* s, kvt_entry* out) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  const size_t n = s->n;
  std::vector<int> tier(n), meth(n);
  std::vector<double> ratio(n);
  std::vector<long long> orig(n), freq(n), last(n), seq(n);
  cudaStream_t st = s->h->stream;
  if (n) {
    KVT_CUDA_TRY(cudaMemcpyAsync(tier.data(), s->d.tier, 4 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(meth.data(), s->d.meth, 4 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(ratio.data(), s->d.ratio, 8 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(orig.data(), s->d.orig, 8 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(freq.data(), s->d.freq, 8 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(last.data(), s->d.last, 8 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaMemcpyAsync(seq.data(), s->d.seq, 8 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaStreamSynchronize(st));
  }
  for (size_t c = 0; c < n; ++c) {
    kvt_entry& e = out[c];
    std::memset(&e, 0, sizeof e);
    e.tier_index = tier[c];
    if (tier[c] < 0) continue;
    e.method = meth[c];
    e.ratio = ratio[c];
    e.original_size_bytes = orig[c];
    e.frequency = freq[c];
    e.last_access = last[c];
    e.seq = seq[c];
  }
  return KVT_OK;
}

extern "C" int kvt_store_actions(kvt_store* s, kvt_action* out, int64_t n) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  Ctl c;
  int rc = store_fetch_ctl(s, &c);
  if (rc) return rc;
  if (n > c.n_act) n = c.n_act;
  if (n > 0) {
    KVT_CUDA_TRY(cudaMemcpyAsync(out, s->act, sizeof(kvt_action) * n, cudaMemcpyDeviceToHost, s->h->stream));
    KVT_CUDA_TRY(cudaStreamSynchronize(s->h->stream));
  }
  return KVT_OK;
}

// Make the store's candidate tables and resident caches current for
// (profiles, space, params, rule).
static int prepare(kvt_store* s, const kvt_pset* p, const kvt_space* space, const kvt_params* params, int rule,
                   StepCtx* X) {
  DevSpace S;
  int rc;
  if ((rc = resolve_space(space, &S))) return rc;
  if (p->dev.M != S.M) return set_error(KVT_EINVAL, "profile set / space method count mismatch");
  if (p->dev.n != s->n) return set_error(KVT_EINVAL, "profile set and store disagree on the context count");
  s->S = S;
  s->has_space = true;
  uint64_t key = fnv(&S, sizeof S);
  key = fnv(&p->id, sizeof p->id, key);
  key = fnv(&params->alpha, sizeof(double), key);
  uint64_t tkey = fnv(&rule, sizeof rule, key);
  cudaStream_t st = s->h->stream;
  const size_t n = std::max(1, s->n), R = S.R, MR = S.M * S.R, TMR = s->TT.T * MR;
  if (tkey != s->tkey) {
    auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t b_size = align(n * R * 8), b_q = align(n * MR * 8), b_v = align(n * MR), b_u = align(n * TMR * 8),
                 b_best = align(n * sizeof(kvt_best));
    const size_t need = b_size + b_q + b_v + b_u + b_best;
    if (need > s->tbytes) {
      cudaFree(s->tbuf);
      s->tbuf = nullptr;
      s->tbytes = 0;
      KVT_CUDA_TRY(cudaMalloc(&s->tbuf, need));
      s->tbytes = need;
    }
    char* b = static_cast<char*>(s->tbuf);
    s->tb = Tables{reinterpret_cast<long long*>(b), reinterpret_cast<double*>(b + b_size),
                   reinterpret_cast<unsigned char*>(b + b_size + b_q), nullptr,
                   reinterpret_cast<double*>(b + b_size + b_q + b_v),
                   reinterpret_cast<kvt_best*>(b + b_size + b_q + b_v + b_u)};
    if ((rc = launch_score(s->h, p->dev, S, s->TT, params->alpha, rule, s->tb))) return rc;
    s->tkey = tkey;
  }
  X->st = s->d;
  X->P = p->dev;
  X->S = S;
  X->alpha = params->alpha;
  X->tb = s->tb;
  if (s->cache_dirty || s->cache_key != key) {
    // errcount reset + per-resident cache + trees bottom-up
    KVT_CUDA_TRY(cudaMemsetAsync(s->d.ctl->errcount, 0, sizeof(int) * KVT_MAX_TIERS, st));
    if (s->n) {
      k_rebuild_cache<<<(s->n * 32 + 127) / 128, 128, 0, st>>>(*X);
      s->h->launches++;
      for (int l = 0; l < s->d.nlev; ++l) {
        dim3 grid((s->d.lvl_size[l] * 32 + 127) / 128, s->TT.T);
        k_tree_level<<<grid, 128, 0, st>>>(s->d, l, 0);
        s->h->launches++;
      }
    }
    KVT_CUDA_TRY(cudaGetLastError());
    s->cache_dirty = false;
    s->cache_key = key;
  }
  return KVT_OK;
}

// Run the persistent greedy over `n_ops` ops already staged on the device,
// growing the action buffer when the kernel asks for it.
static int run_greedy(kvt_store* s, StepCtx& X, Ops ops, long long n_ops, int64_t* n_actions, int64_t* n_done) {
  cudaStream_t st = s->h->stream;
  Ctl init{};
  {
    Ctl cur;
    int rc = store_fetch_ctl(s, &cur);
    if (rc) return rc;
    init = cur;
  }
  init.n_act = 0;
  init.n_ops = n_ops;
  init.resume_op = 0;
  init.in_resolve = n_ops < 0 ? 1 : 0;  // resolve-only call
  if (n_ops < 0) init.n_ops = 1;        // one pseudo op: the resolve
  init.status = ST_OK;
  long long need = std::max<long long>(4096, 8 * (init.n_ops + 16));
  if (need > s->cap_act) {
    cudaFree(s->act);
    s->act = nullptr;
    KVT_CUDA_TRY(cudaMalloc(&s->act, sizeof(kvt_action) * need));
    s->cap_act = need;
    s->d.act = s->act;
  }
  init.cap_act = s->cap_act;
  KVT_CUDA_TRY(cudaMemcpyAsync(s->d.ctl, &init, sizeof(Ctl), cudaMemcpyHostToDevice, st));
  Ctl c;
  while (true) {
    X.st = s->d;
    k_greedy<<<1, 32, 0, st>>>(X, ops);
    s->h->launches++;
    KVT_CUDA_TRY(cudaGetLastError());
    int rc = store_fetch_ctl(s, &c);
    if (rc) return rc;
    if (c.status != ST_NEED_SPACE) break;
    const long long ncap = s->cap_act * 2;
    kvt_action* na = nullptr;
    KVT_CUDA_TRY(cudaMalloc(&na, sizeof(kvt_action) * ncap));
    KVT_CUDA_TRY(cudaMemcpyAsync(na, s->act, sizeof(kvt_action) * c.n_act, cudaMemcpyDeviceToDevice, st));
    KVT_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFree(s->act);
    s->act = na;
    s->cap_act = ncap;
    s->d.act = na;
    c.cap_act = ncap;
    c.status = ST_OK;
    KVT_CUDA_TRY(cudaMemcpyAsync(s->d.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
  }
  *n_actions = c.n_act;
  if (n_done) *n_done = n_ops < 0 ? 0 : (c.in_resolve ? c.resume_op : c.resume_op);
  return store_status_error(s, c);
}

static int stage_ops(kvt_store* s, const int32_t* ctx, const int64_t* freq, const int64_t* stamp, long long n) {
  if (n > s->ops_cap) {
    cudaFree(s->ops_buf);
    cudaFree(s->ops_l);
    s->ops_buf = nullptr;
    s->ops_l = nullptr;
    KVT_CUDA_TRY(cudaMalloc(&s->ops_buf, 4 * n));
    KVT_CUDA_TRY(cudaMalloc(&s->ops_l, 16 * n));
    s->ops_cap = n;
  }
  cudaStream_t st = s->h->stream;
  for (long long i = 0; i < n; ++i)
    if (ctx[i] < 0 || ctx[i] >= s->n) return set_error(KVT_EINVAL, "context index out of range");
  KVT_CUDA_TRY(cudaMemcpyAsync(s->ops_buf, ctx, 4 * n, cudaMemcpyHostToDevice, st));
  if (freq) KVT_CUDA_TRY(cudaMemcpyAsync(s->ops_l, freq, 8 * n, cudaMemcpyHostToDevice, st));
  else KVT_CUDA_TRY(cudaMemsetAsync(s->ops_l, 0, 8 * n, st));
  if (stamp) KVT_CUDA_TRY(cudaMemcpyAsync(s->ops_l + n, stamp, 8 * n, cudaMemcpyHostToDevice, st));
  else KVT_CUDA_TRY(cudaMemsetAsync(s->ops_l + n, 0, 8 * n, st));
  return KVT_OK;
}

extern "C" int kvt_insert_joint(kvt_store* s, const kvt_pset* p, const kvt_space* space, const kvt_params* params,
                                int32_t rule, const int32_t* ctx, const int64_t* frequency, const int64_t* stamp,
                                int64_t n_ops, int64_t* n_actions, int64_t* n_done) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  *n_actions = 0;
  *n_done = 0;
  StepCtx X;
  int rc;
  if ((rc = prepare(s, p, space, params, rule, &X))) return rc;
  if (n_ops <= 0) return KVT_OK;
  if ((rc = stage_ops(s, ctx, frequency, stamp, n_ops))) return rc;
  Ops ops{s->ops_buf, s->ops_l, s->ops_l + n_ops};
  return run_greedy(s, X, ops, n_ops, n_actions, n_done);
}

extern "C" int kvt_resolve_overflow(kvt_store* s, const kvt_pset* p, const kvt_space* space,
                                    const kvt_params* params, int64_t* n_actions) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  StepCtx X;
  int rc;
  *n_actions = 0;
  if ((rc = prepare(s, p, space, params, KVT_RULE_UTILITY, &X))) return rc;
  Ops ops{s->d.saved, nullptr, nullptr};
  return run_greedy(s, X, ops, -1, n_actions, nullptr);
}

extern "C" int kvt_least_drop_update(kvt_store* s, const kvt_pset* p, const kvt_space* space,
                                     const kvt_params* params, int32_t tier_index, kvt_update* out) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  StepCtx X;
  int rc;
  if (tier_index < 0 || tier_index >= s->TT.T) return set_error(KVT_EINVAL, "tier index out of range");
  if ((rc = prepare(s, p, space, params, KVT_RULE_UTILITY, &X))) return rc;
  kvt_update* d_u = nullptr;
  KVT_CUDA_TRY(cudaMallocAsync(&d_u, sizeof(kvt_update), s->h->stream));
  if (s->TT.unlimited[tier_index] && s->n) {
    // the greedy never pops the unlimited bottom tier, so it does not keep
    // that tier's tree current: rebuild it from the per-resident caches
    for (int l = 0; l < s->d.nlev; ++l) {
      dim3 grid((s->d.lvl_size[l] * 32 + 127) / 128, 1);
      k_tree_level<<<grid, 128, 0, s->h->stream>>>(s->d, l, tier_index);
      s->h->launches++;
    }
  }
  k_ld_query<<<1, 1, 0, s->h->stream>>>(X, tier_index, d_u);
  s->h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  KVT_CUDA_TRY(cudaMemcpyAsync(out, d_u, sizeof(kvt_update), cudaMemcpyDeviceToHost, s->h->stream));
  KVT_CUDA_TRY(cudaFreeAsync(d_u, s->h->stream));
  Ctl c;
  if ((rc = store_fetch_ctl(s, &c))) return rc;
  return store_status_error(s, c);
}

// Stable LSD radix sort of (u64 key, int value) pairs, ascending, in one
// 1024-thread CTA (rearrange / placement_utility: one sort of <= the store's
// contexts per call, off the bench's hot loop). Eight 8-bit passes ping-pong
// between the two buffers; a pass whose digit is the same for every key is
// skipped. Per 1,024-element tile: a thread's rank among equal digits of
// its warp (__match_any_sync), per-(warp, digit) counts prefix-summed over
// the warps in smem, plus the digit's running base over earlier tiles —
// stable by construction. The sorted pairs end in (k_out, v_out); k_in /
// v_in are scratch.
constexpr int kSortT = 1024;
__global__ void __launch_bounds__(kSortT) k_sort_pairs(unsigned long long* __restrict__ k_in, int* __restrict__ v_in,
                                                       unsigned long long* __restrict__ k_out,
                                                       int* __restrict__ v_out, int n) {
  __shared__ int wcnt[kSortT / 32][256];
  __shared__ int base[256], tot[256];
  __shared__ int skip;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long* sk = k_in;
  int* sv = v_in;
  unsigned long long* dk = k_out;
  int* dv = v_out;
  for (int pass = 0; pass < 8; ++pass) {
    const int sh = 8 * pass;
    if (tid < 256) base[tid] = 0;
    if (tid == 0) skip = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kSortT) atomicAdd(&base[static_cast<int>((sk[i] >> sh) & 255)], 1);
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 256 digit counts: 8 bins per lane + a warp scan
      int c[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = base[8 * lane + j];
        if (c[j] == n) skip = 1;  // every key has this digit: the pass is the identity
        sum += c[j];
      }
      int incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      int run = incl - sum;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        base[8 * lane + j] = run;
        run += c[j];
      }
    }
    __syncthreads();
    if (skip) continue;  // block-uniform
    for (int t0 = 0; t0 < n; t0 += kSortT) {
      const int i = t0 + tid;
      const bool live = i < n;
      const unsigned long long key = live ? sk[i] : 0ull;
      const int val = live ? sv[i] : 0;
      const int d = live ? static_cast<int>((key >> sh) & 255) : 256;
      for (int j = tid; j < (kSortT / 32) * 256; j += kSortT) (&wcnt[0][0])[j] = 0;
      __syncthreads();
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int lower = __popc(peers & ((1u << lane) - 1u));
      if (live && lower == 0) wcnt[warp][d] = __popc(peers);
      __syncthreads();
      if (tid < 256) {  // per digit: exclusive prefix over the warps, and the tile's total
        int acc = 0;
        for (int w = 0; w < kSortT / 32; ++w) {
          const int c = wcnt[w][tid];
          wcnt[w][tid] = acc;
          acc += c;
        }
        tot[tid] = acc;
      }
      __syncthreads();
      if (live) {
        const int pos = base[d] + wcnt[warp][d] + lower;
        dk[pos] = key;
        dv[pos] = val;
      }
      __syncthreads();
      if (tid < 256) base[tid] += tot[tid];
      __syncthreads();
    }
    unsigned long long* tk = sk;
    sk = dk;
    dk = tk;
    int* tv = sv;
    sv = dv;
    dv = tv;
    __syncthreads();  // this pass's scatter visible to the whole CTA before the next reads it
  }
  if (sk != k_out)  // the result is in the scratch pair: copy it out
    for (int i = tid; i < n; i += kSortT) {
      k_out[i] = sk[i];
      v_out[i] = sv[i];
    }
}

// keys/vals double buffers for the radix sorts (n each)
static int sort_pairs(kvt_store* s, unsigned long long* k_in, unsigned long long* k_out, int* v_in, int* v_out,
                      int n) {
  k_sort_pairs<<<1, kSortT, 0, s->h->stream>>>(k_in, v_in, k_out, v_out, n);
  s->h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  return KVT_OK;
}

extern "C" int kvt_rearrange(kvt_store* s, const kvt_pset* p, const kvt_space* space, const kvt_params* params,
                             int32_t rule, int64_t* n_actions) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  StepCtx X;
  int rc;
  *n_actions = 0;
  if ((rc = prepare(s, p, space, params, rule, &X))) return rc;
  if (s->n == 0) return KVT_OK;
  cudaStream_t st = s->h->stream;
  const size_t n = s->n;
  char* tmp = nullptr;
  KVT_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * 24 + 1024, st));
  auto* k_in = reinterpret_cast<unsigned long long*>(tmp);
  auto* k_out = k_in + n;
  auto* v_in = reinterpret_cast<int*>(k_out + n);
  Ctl c;
  if ((rc = store_fetch_ctl(s, &c))) return rc;
  c.n_saved = 0;
  c.status = ST_OK;
  KVT_CUDA_TRY(cudaMemcpyAsync(s->d.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
  k_rearrange_keys<<<(s->n + 255) / 256, 256, 0, st>>>(s->d, s->tb.best, k_in, v_in);
  s->h->launches++;
  KVT_CUDA_TRY(cudaGetLastError());
  if ((rc = sort_pairs(s, k_in, k_out, v_in, s->d.saved, s->n))) return rc;
  if ((rc = store_fetch_ctl(s, &c))) return rc;
  cudaFreeAsync(tmp, st);
  if (c.status != ST_OK) return store_status_error(s, c);
  const int n_saved = c.n_saved;
  // store.clear() then re-insert in saved order, keeping access stats
  k_clear<<<(s->n + 255) / 256 + 1, 256, 0, st>>>(s->d);
  s->h->launches++;
  KVT_CUDA_TRY(cudaMemsetAsync(s->d.tree, 0xff, 4 * static_cast<size_t>(s->d.tree_stride) * s->TT.T, st));
  KVT_CUDA_TRY(cudaMemsetAsync(s->d.tkey, 0xff, sizeof(ulonglong2) * static_cast<size_t>(s->d.tree_stride) * s->TT.T, st));
  KVT_CUDA_TRY(cudaGetLastError());
  Ops ops{s->d.saved, nullptr, nullptr};
  if (n_saved == 0) return KVT_OK;
  return run_greedy(s, X, ops, n_saved, n_actions, nullptr);
}

extern "C" int kvt_placement_utility(kvt_store* s, const kvt_pset* p, const kvt_space* space,
                                     const kvt_params* params, double* out) {
  KVT_ON_DEVICE((s ? s->h : nullptr));
  StepCtx X;
  int rc;
  if ((rc = prepare(s, p, space, params, KVT_RULE_UTILITY, &X))) return rc;
  *out = 0.0;
  if (s->n == 0) return KVT_OK;
  cudaStream_t st = s->h->stream;
  const size_t n = s->n;
  char* tmp = nullptr;
  KVT_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * 36 + 2048, st));
  auto* term = reinterpret_cast<double*>(tmp);
  auto* k_in = reinterpret_cast<unsigned long long*>(term + n);
  auto* k_out = k_in + n;
  auto* v_in = reinterpret_cast<int*>(k_out + n);
  auto* v_out = v_in + n;
  auto* bad = v_out + n;
  auto* d_out = reinterpret_cast<double*>(bad + 2);
  KVT_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
  k_util_terms<<<(s->n + 255) / 256, 256, 0, st>>>(X, term, k_in, v_in, bad);
  s->h->launches++;
  if ((rc = sort_pairs(s, k_in, k_out, v_in, v_out, s->n))) return rc;
  Ctl c;
  if ((rc = store_fetch_ctl(s, &c))) return rc;
  int n_res = 0;
  {
    // number of residents = contexts with a tier; count on host from keys
    std::vector<unsigned long long> keys(n);
    KVT_CUDA_TRY(cudaMemcpyAsync(keys.data(), k_out, 8 * n, cudaMemcpyDeviceToHost, st));
    KVT_CUDA_TRY(cudaStreamSynchronize(st));
    while (n_res < s->n && keys[n_res] != ~0ull) ++n_res;
  }
  k_util_sum<<<1, 1, 0, st>>>(term, v_out, n_res, d_out);
  s->h->launches++;
  int h_bad = 0;
  KVT_CUDA_TRY(cudaMemcpyAsync(out, d_out, sizeof(double), cudaMemcpyDeviceToHost, st));
  KVT_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  KVT_CUDA_TRY(cudaFreeAsync(tmp, st));
  KVT_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_bad) return set_error(KVT_EVALIDATION, "resident " + std::to_string(h_bad - 1) +
                                                   " has a configuration its profile cannot score");
  return KVT_OK;
}

// ------------------------------------------------------------ tier moves
// Tier-move executor (include/kvt_b200.h). Each handle owns
// two copy streams per direction; a batch is split into <= 8 MiB pieces
// dealt round-robin over the streams of its direction, fenced after the
// handle's stream (input ready) and joined back into it (completion).
namespace {
constexpr int64_t kMovePiece = 8LL << 20;

int move_streams(kvt_handle* h) {  // the handle's copy streams, created on first use
  if (h->move_s[0]) return KVT_OK;
  for (int i = 0; i < 4; ++i) {
    KVT_CUDA_TRY(cudaStreamCreateWithFlags(&h->move_s[i], cudaStreamNonBlocking));
    KVT_CUDA_TRY(cudaEventCreateWithFlags(&h->move_done[i], cudaEventDisableTiming));
  }
  KVT_CUDA_TRY(cudaEventCreateWithFlags(&h->move_start, cudaEventDisableTiming));
  return KVT_OK;
}
}  // namespace

extern "C" int kvt_tier_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return set_error(KVT_EINVAL, "bad host arena request");
  *out = nullptr;
  KVT_CUDA_TRY(cudaHostAlloc(out, static_cast<size_t>(bytes > 0 ? bytes : 1), cudaHostAllocDefault));
  return KVT_OK;
}

extern "C" int kvt_tier_host_free(void* p) {
  if (p) KVT_CUDA_TRY(cudaFreeHost(p));
  return KVT_OK;
}

extern "C" int kvt_tier_moves(kvt_handle* h, const kvt_move* moves, int64_t n) {
  if (!h || (n > 0 && !moves)) return set_error(KVT_EINVAL, "null argument");
  if (n <= 0) return KVT_OK;
  DeviceGuard dg(h->device);
  int rc;
  if ((rc = move_streams(h))) return rc;
  KVT_CUDA_TRY(cudaEventRecord(h->move_start, h->stream));
  bool used[4] = {false, false, false, false};
  int next[2] = {0, 0};  // round-robin per direction class (0: to host, 1: to device)
  for (int64_t i = 0; i < n; ++i) {
    const kvt_move& mv = moves[i];
    if (mv.bytes < 0 || (mv.bytes > 0 && (!mv.src || !mv.dst)) || mv.kind < 0 || mv.kind > KVT_MOVE_H2H)
      return set_error(KVT_EINVAL, "bad move " + std::to_string(i));
    static const cudaMemcpyKind kinds[4] = {cudaMemcpyDeviceToHost, cudaMemcpyHostToDevice, cudaMemcpyDeviceToDevice,
                                            cudaMemcpyHostToHost};
    const int cls = (mv.kind == KVT_MOVE_H2D || mv.kind == KVT_MOVE_D2D) ? 1 : 0;
    for (int64_t off = 0; off < mv.bytes; off += kMovePiece) {
      const int si = cls * 2 + next[cls];
      next[cls] ^= 1;
      if (!used[si]) {
        KVT_CUDA_TRY(cudaStreamWaitEvent(h->move_s[si], h->move_start, 0));
        used[si] = true;
      }
      const size_t len = static_cast<size_t>(std::min(kMovePiece, mv.bytes - off));
      KVT_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(mv.dst) + off, static_cast<const char*>(mv.src) + off, len,
                                   kinds[mv.kind], h->move_s[si]));
    }
  }
  for (int i = 0; i < 4; ++i)
    if (used[i]) {
      KVT_CUDA_TRY(cudaEventRecord(h->move_done[i], h->move_s[i]));
      KVT_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->move_done[i], 0));
    }
  return KVT_OK;
}
