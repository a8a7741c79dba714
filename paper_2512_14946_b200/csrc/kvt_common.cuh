// Shared device/host helpers of libkvt_b200.so.
//
// All placement arithmetic is FP64 written with explicit round-to-nearest
// intrinsics (__dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn) in the reference's
// evaluation order, so nvcc cannot contract it into FMAs (one
// contraction changes the reference's results bit-for-bit). The file is also
// compiled with -fmad=false as a second guard.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "kvt_b200.h"

namespace kvt {

constexpr double kGridEps = 1e-9;  // proj/src/quality.cpp:16
constexpr int kWarp = 32;

// Space / tiers as kernel parameters (by value, a few hundred bytes).
struct DevSpace {
  int M, R;
  double ratio[KVT_MAX_RATIOS];   // CandidateSpace order (descending)
  double ovh[KVT_MAX_METHODS];    // decompression overhead, s/byte
  int name_rank[KVT_MAX_METHODS]; // byte-lexicographic rank of method name
};

struct DevTiers {
  int T;
  int id[KVT_MAX_TIERS];
  int unlimited[KVT_MAX_TIERS];
  long long cap[KVT_MAX_TIERS];
  double bw[KVT_MAX_TIERS];
  double lat[KVT_MAX_TIERS];
};

// Device copy of a kvt_profiles set.
struct DevProfiles {
  int n, M;
  const long long* orig;
  const double* freq;
  const int* goff;
  const double* grid;
  const double* qual;
  const unsigned char* has;
};

// compressed_size proj/src/core.cpp:72-84 (ratio already validated in (0,1])
__host__ __device__ inline long long csize(long long orig, double ratio) {
#ifdef __CUDA_ARCH__
  const double scaled = __dmul_rn(static_cast<double>(orig), ratio);
  const long long b = static_cast<long long>(floor(__dadd_rn(scaled, 0.5)));
#else
  const double scaled = static_cast<double>(orig) * ratio;
  const long long b = static_cast<long long>(floor(scaled + 0.5));
#endif
  return b > 1 ? b : 1;
}

#ifdef __CUDACC__
// load_time proj/src/utility.cpp:51-59: (lat + s/bw) + s*ovh
__device__ __forceinline__ double load_time(long long size, double lat, double bw, double ovh) {
  const double s = static_cast<double>(size);
  return __dadd_rn(__dadd_rn(lat, __ddiv_rn(s, bw)), __dmul_rn(s, ovh));
}

// utility_score proj/src/utility.cpp:61-63: (alpha*q - ttft)*f
__device__ __forceinline__ double utility_score(double q, double ttft, double f, double alpha) {
  return __dmul_rn(__dsub_rn(__dmul_rn(alpha, q), ttft), f);
}

// scorable proj/src/utility.cpp:13-17
__device__ __forceinline__ bool scorable(const DevProfiles& p, int c, int m, double ratio) {
  if (!p.has[static_cast<size_t>(c) * p.M + m]) return false;
  return ratio >= __dsub_rn(p.grid[p.goff[c]], kGridEps);
}

// quality_of proj/src/quality.cpp:86-113 for a scorable (c, m, ratio);
// returns false if the reference would throw.
__device__ inline bool quality_of(const DevProfiles& p, int c, int m, double ratio, double* out) {
  if (!(ratio > 0.0) || ratio > __dadd_rn(1.0, kGridEps)) return false;
  if (!p.has[static_cast<size_t>(c) * p.M + m]) return false;
  const int g0 = p.goff[c], len = p.goff[c + 1] - g0;
  const double* grid = p.grid + g0;
  const double* val = p.qual + static_cast<size_t>(g0) * p.M + static_cast<size_t>(m) * len;
  if (ratio < __dsub_rn(grid[0], kGridEps)) return false;
  const double key = __dsub_rn(ratio, kGridEps);
  int i = 0;  // std::lower_bound
  while (i < len && grid[i] < key) ++i;
  if (i >= len) i = len - 1;
  if (fabs(__dsub_rn(grid[i], ratio)) <= kGridEps || i == 0) {
    *out = val[i];
    return true;
  }
  const double x0 = grid[i - 1], x1 = grid[i];
  const double y0 = val[i - 1], y1 = val[i];
  const double t = __ddiv_rn(__dsub_rn(ratio, x0), __dsub_rn(x1, x0));
  *out = __dadd_rn(y0, __dmul_rn(t, __dsub_rn(y1, y0)));
  return true;
}
#endif

// ------------------------------------------------------------ host helpers
}  // namespace kvt

// Handle: device, stream, scratch, and a launch counter (bench evidence).
struct kvt_handle {
  ~kvt_handle();
  int device = 0;
  cudaStream_t stream = nullptr;
  long long launches = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // snapkv Q8 tiles depend only on (L, H, W, G, q_seed), not on the KV
  // chunk: generated once per key and reused by every chunk of that shape
  void* snapq = nullptr;
  size_t snapq_bytes = 0;
  unsigned long long snapq_key[5] = {0, 0, 0, 0, 0};
  void* snape = nullptr;  // snapkv E scratch slots for prefixes beyond 8192 tokens
  size_t snape_bytes = 0;
  // tier-move executor: two copy streams per direction (d2h x2, h2d x2),
  // created on first use, destroyed with the handle
  cudaStream_t move_s[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t move_start = nullptr, move_done[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace kvt {
struct Error {
  int code;
  std::string msg;
};

int set_error(int code, const std::string& msg);

// Per-device facts and one-time kernel attributes. The ABI lets one process
// drive several devices (kvt_create(device, ...)) from several threads (the
// reference's `compare --jobs`), so nothing here is a plain static: every
// cache is keyed by device ordinal and guarded by a mutex.
int device_sms(int dev);
int device_smem_optin(int dev);
// cudaFuncSetAttribute(fn, a, value) on device `dev` (current device must be
// dev, see DeviceGuard), issued once per (fn, a, dev, value)
cudaError_t func_attr(const void* fn, int dev, cudaFuncAttribute a, int value);
// value cached per (fn, dev, key); compute() runs once (occupancy queries)
int cached_per_device(const void* fn, int dev, long long key, int (*compute)(void*), void* arg);

// Makes h->device current for the duration of an ABI call and restores the
// caller's device afterwards (no cudaSetDevice side effect leaks out).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

#define KVT_ON_DEVICE(hp)                                                      \
  if (!(hp)) return ::kvt::set_error(KVT_EINVAL, "null handle");               \
  ::kvt::DeviceGuard kvt_dg__((hp)->device)

#define KVT_CUDA_TRY(expr)                                                     \
  do {                                                                         \
    cudaError_t e__ = (expr);                                                  \
    if (e__ != cudaSuccess)                                                    \
      return ::kvt::set_error(KVT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

}  // namespace kvt
