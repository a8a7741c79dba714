// kvtier -> libkvt_b200.so drop-in shim.
//
// Re-implements the hot-path free functions of the reference's public C++
// API (proj/include/kvtier/utility.hpp, proj/include/kvtier/placement.hpp)
// on top of the C ABI in include/kvt_b200.h, so an unmodified kvtier build
// (Replayer, policies, CLI, tests) runs its candidate scoring and
// least-utility-drop placement on the B200 kernels. It is the binding a
// reference maintainer adds; see INTEGRATION.md for the two ways to link it
// (replace utility.cpp/placement.cpp at link time, or ELF interposition in
// front of an -fPIC libkvtier, which is what oracle/Makefile's
// `acceptance-b200` target builds to run the reference's own acceptance
// gate on the GPU).
//
// Functions provided (reference declaration -> C ABI call):
//   all_candidates      utility.hpp:79-82   -> kvt_score_candidates
//   best_config         utility.hpp:96-99   -> kvt_best_config
//   least_drop_update   placement.hpp:87-90 -> kvt_least_drop_update
//   resolve_overflow    placement.hpp:94-96 -> kvt_resolve_overflow
//   insert_joint        placement.hpp:101-106 -> kvt_insert_joint
//   rearrange           placement.hpp:111-114 -> kvt_rearrange
//   placement_utility   placement.hpp:117-118 -> kvt_placement_utility
//
// Each call mirrors the caller's StoreState into a device store, runs the
// op, and replays the returned action list onto the StoreState through its
// public mutators (add / remove / reconfigure), so the host object ends in
// exactly the state the reference would leave it in (the action lists are
// bit-identical, tests/test_gpu_placement.py). This per-call mirror is
// O(residents) host work: right for a drop-in, not for a hot serving loop,
// which keeps the kvt_store resident across calls (bench.py does).
// Status codes map back to the reference's exceptions: KVT_EVALIDATION ->
// kvtier::ValidationError, KVT_ETRACE -> kvtier::TraceError, anything else
// -> std::runtime_error (proj/include/kvtier/core.hpp:18-24).
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kvt_b200.h"
#include "kvtier/core.hpp"
#include "kvtier/placement.hpp"
#include "kvtier/quality.hpp"
#include "kvtier/utility.hpp"

namespace kvtier {
namespace {

// KVT_SHIM_TRACE=1: report at exit how many reference calls the shim served
// (the drop-in test uses it to prove the interposition took effect).
struct CallCount {
  std::atomic<long> n{0};  // worker threads of `compare --jobs` call concurrently
  ~CallCount() {
    if (std::getenv("KVT_SHIM_TRACE")) std::fprintf(stderr, "kvt_b200 shim: %ld kvtier calls served\n", n.load());
  }
} g_calls;

void check(int rc) {
  if (rc == KVT_OK) return;
  const std::string msg = kvt_last_error();
  if (rc == KVT_EVALIDATION) throw ValidationError(msg);
  if (rc == KVT_ETRACE) throw TraceError(msg);
  throw std::runtime_error("kvt_b200: " + msg);
}

// One handle per thread (the reference runs independent stores on worker
// threads under `compare --jobs`, proj/tools/kvtier_main.cpp:206-235).
kvt_handle* handle() {
  g_calls.n.fetch_add(1, std::memory_order_relaxed);
  struct Owner {
    kvt_handle* h = nullptr;
    ~Owner() {
      if (h) kvt_destroy(h);
    }
  };
  thread_local Owner o;
  if (!o.h) check(kvt_create(0, nullptr, &o.h));
  return o.h;
}

// CandidateSpace / MethodSet as the ABI's kvt_space (names kept alive here).
struct Space {
  std::vector<std::string> names;
  std::vector<const char*> cnames;
  std::vector<double> overhead, ratios;
  kvt_space s{};

  Space(const MethodSet& methods, std::vector<double> grid) : ratios(std::move(grid)) {
    for (const auto& m : methods.methods()) {
      names.push_back(m.name);
      overhead.push_back(m.decompression_overhead);
    }
    for (const auto& n : names) cnames.push_back(n.c_str());
    s.n_methods = static_cast<int32_t>(names.size());
    s.method_names = cnames.data();
    s.decompression_overhead = overhead.data();
    s.n_ratios = static_cast<int32_t>(ratios.size());
    s.ratios = ratios.data();
  }
  explicit Space(const CandidateSpace& cs) : Space(cs.methods(), cs.ratios()) {}

  int32_t method(const std::string& name) const {
    for (size_t i = 0; i < names.size(); ++i)
      if (names[i] == name) return static_cast<int32_t>(i);
    throw ValidationError("unknown compression method " + name);
  }
};

std::vector<kvt_tier> abi_tiers(const std::vector<TierSpec>& tiers) {
  std::vector<kvt_tier> out;
  for (const auto& t : tiers) {
    kvt_tier k{};
    k.tier_id = t.tier_id;
    k.unlimited = t.unlimited() ? 1 : 0;
    k.capacity_bytes = t.capacity_bytes.value_or(0);
    k.read_bandwidth = t.read_bandwidth;
    k.fixed_access_latency = t.fixed_access_latency;
    out.push_back(k);
  }
  return out;
}

// Profiles in ProfileMap order (byte-lexicographic ContextId = ABI context
// index), quality rows per space method.
struct Profiles {
  std::vector<const ContextProfile*> by_index;
  std::vector<int64_t> orig;
  std::vector<double> freq, grid, qual;
  std::vector<int32_t> goff{0};
  std::vector<uint8_t> has;
  kvt_pset* p = nullptr;

  Profiles(const std::vector<const ContextProfile*>& ps, const Space& sp) : by_index(ps) {
    const size_t M = sp.names.size();
    for (const ContextProfile* pr : ps) {
      orig.push_back(pr->original_size_bytes);
      freq.push_back(pr->frequency);
      const size_t len = pr->ratio_grid.size();
      grid.insert(grid.end(), pr->ratio_grid.begin(), pr->ratio_grid.end());
      for (size_t m = 0; m < M; ++m) {
        auto it = pr->quality_table.find(sp.names[m]);
        const bool ok = it != pr->quality_table.end() && it->second.size() == len;
        has.push_back(ok ? 1 : 0);
        for (size_t i = 0; i < len; ++i) qual.push_back(ok ? it->second[i] : 0.0);
      }
      goff.push_back(static_cast<int32_t>(grid.size()));
    }
    kvt_profiles raw{};
    raw.n_ctx = static_cast<int32_t>(ps.size());
    raw.n_methods = static_cast<int32_t>(M);
    raw.original_size_bytes = orig.data();
    raw.frequency = freq.data();
    raw.grid_offset = goff.data();
    raw.grid = grid.data();
    raw.quality = qual.data();
    raw.has_method = has.data();
    check(kvt_pset_create(handle(), &raw, &p));
  }
  ~Profiles() { kvt_pset_destroy(p); }
  Profiles(const Profiles&) = delete;
  Profiles& operator=(const Profiles&) = delete;
};

std::vector<const ContextProfile*> ordered(const ProfileMap& profiles) {
  std::vector<const ContextProfile*> v;
  for (const auto& kv : profiles) v.push_back(&kv.second);
  return v;
}

int32_t ctx_index(const ProfileMap& profiles, const ContextId& id) {
  auto it = profiles.find(id);
  if (it == profiles.end()) throw ValidationError("no profile for context " + id);
  return static_cast<int32_t>(std::distance(profiles.begin(), it));
}

int tier_index_of_id(const std::vector<TierSpec>& tiers, int tier_id) {
  for (size_t i = 0; i < tiers.size(); ++i)
    if (tiers[i].tier_id == tier_id) return static_cast<int>(i);
  throw ValidationError("unknown tier id " + std::to_string(tier_id));
}

// Device mirror of a StoreState: residents added tier by tier in arrival
// order, which is the order the device store keeps inside a tier.
struct Mirror {
  kvt_store* s = nullptr;
  Mirror(const StoreState& store, const ProfileMap& profiles, const Space& sp) {
    const auto tiers = abi_tiers(store.tiers());
    check(kvt_store_create(handle(), tiers.data(), static_cast<int32_t>(tiers.size()),
                           static_cast<int32_t>(profiles.size()), &s));
    check(kvt_store_bind_space(s, &sp.s));
    for (size_t ti = 0; ti < store.tier_count(); ++ti)
      for (const CacheEntry& e : store.residents(ti)) {
        kvt_entry k{};
        k.tier_index = static_cast<int32_t>(ti);
        k.method = sp.method(e.config.method);
        k.ratio = e.config.ratio;
        k.original_size_bytes = e.original_size_bytes;
        k.frequency = e.frequency;
        k.last_access = e.last_access;
        check(kvt_store_add(s, ctx_index(profiles, e.context), &k));
      }
  }
  ~Mirror() { kvt_store_destroy(s); }
  Mirror(const Mirror&) = delete;
  Mirror& operator=(const Mirror&) = delete;

  std::vector<kvt_action> actions(int64_t n) {
    std::vector<kvt_action> a(static_cast<size_t>(n));
    if (n) check(kvt_store_actions(s, a.data(), n));
    return a;
  }
};

PlacementAction to_action(const kvt_action& a, const Profiles& P, const Space& sp) {
  PlacementAction out;
  out.kind = a.kind == KVT_INSERT ? PlacementAction::Kind::Insert
             : a.kind == KVT_RECOMPRESS ? PlacementAction::Kind::Recompress
                                        : PlacementAction::Kind::Evict;
  out.context = P.by_index[a.ctx]->context;
  out.tier = a.tier_id;
  out.config = CompressionConfig{sp.names[a.method], a.ratio};
  return out;
}

// Replays device actions onto the host StoreState with the same mutations
// the reference makes (placement.cpp:213-221 for updates, :236-244 for the
// insert). `stats(ctx)` gives (frequency, stamp) for an Insert.
template <class Stats>
void apply(StoreState& store, const std::vector<kvt_action>& acts, const Profiles& P, const Space& sp,
           Stats&& stats, std::vector<PlacementAction>& out) {
  for (const kvt_action& a : acts) {
    const PlacementAction pa = to_action(a, P, sp);
    if (pa.kind == PlacementAction::Kind::Insert) {
      CacheEntry e;
      e.context = pa.context;
      e.original_size_bytes = P.by_index[a.ctx]->original_size_bytes;
      e.config = pa.config;
      e.tier = pa.tier;
      const auto fs = stats(a.ctx);
      e.frequency = fs.first;
      e.last_access = fs.second;
      store.add(std::move(e));
    } else if (pa.kind == PlacementAction::Kind::Recompress) {
      store.reconfigure(pa.context, pa.config);
    } else {
      CacheEntry moved = store.remove(pa.context);
      moved.tier = pa.tier;
      moved.config = pa.config;
      store.add(std::move(moved));
    }
    out.push_back(pa);
  }
}

ConfigCandidate candidate(const ContextProfile& pr, const std::vector<TierSpec>& tiers, int tier_index,
                          const std::string& method, double ratio, int64_t size, double q, double ttft,
                          double u) {
  ConfigCandidate c;
  c.tier_index = tier_index;
  c.tier_id = tiers[static_cast<size_t>(tier_index)].tier_id;
  c.config = CompressionConfig{method, ratio};
  c.size_bytes = size;
  c.quality = q;
  c.ttft = ttft;
  c.frequency = pr.frequency;
  c.utility = u;
  return c;
}

}  // namespace

std::vector<ConfigCandidate> all_candidates(const ContextProfile& profile, const std::vector<TierSpec>& tiers,
                                            const CandidateSpace& space, const UtilityParams& params) {
  const Space sp(space);
  const Profiles P({&profile}, sp);
  const auto kt = abi_tiers(tiers);
  const kvt_params pr{params.alpha};
  const size_t T = kt.size(), M = sp.names.size(), R = space.ratios().size();
  std::vector<int64_t> size(R);
  std::vector<double> q(M * R), ttft(T * M * R), u(T * M * R);
  std::vector<uint8_t> valid(M * R);
  check(kvt_score_candidates(handle(), P.p, kt.data(), static_cast<int32_t>(T), &sp.s, &pr, size.data(), q.data(),
                             valid.data(), ttft.data(), u.data()));
  // enumeration order tier -> method -> ratio (utility.cpp:129-145);
  // space.ratios() is already the sorted, de-duplicated device order
  std::vector<ConfigCandidate> out;
  for (size_t t = 0; t < T; ++t)
    for (size_t m = 0; m < M; ++m)
      for (size_t r = 0; r < R; ++r) {
        if (!valid[m * R + r]) continue;
        const size_t i = (t * M + m) * R + r;
        out.push_back(candidate(profile, tiers, static_cast<int>(t), sp.names[m], space.ratios()[r], size[r],
                                q[m * R + r], ttft[i], u[i]));
      }
  return out;
}

ConfigCandidate best_config(const ContextProfile& profile, const std::vector<TierSpec>& tiers,
                            const CandidateSpace& space, const UtilityParams& params, SelectionRule rule) {
  const Space sp(space);
  const Profiles P({&profile}, sp);
  const auto kt = abi_tiers(tiers);
  const kvt_params pr{params.alpha};
  kvt_best b{};
  check(kvt_best_config(handle(), P.p, kt.data(), static_cast<int32_t>(kt.size()), &sp.s, &pr,
                        rule == SelectionRule::QualityFirst ? KVT_RULE_QUALITY_FIRST : KVT_RULE_UTILITY, &b));
  if (b.status != 0) throw ValidationError("context " + profile.context + " has no scorable configuration");
  return candidate(profile, tiers, b.tier_index, sp.names[b.method], b.ratio, b.size_bytes, b.quality, b.ttft,
                   b.utility);
}

UpdateCandidate least_drop_update(const StoreState& store, std::size_t tier_index, const ProfileMap& profiles,
                                  const CandidateSpace& space, const UtilityParams& params) {
  const Space sp(space);
  const Profiles P(ordered(profiles), sp);
  Mirror mir(store, profiles, sp);
  const kvt_params pr{params.alpha};
  kvt_update u{};
  check(kvt_least_drop_update(mir.s, P.p, &sp.s, &pr, static_cast<int32_t>(tier_index), &u));
  const ContextProfile& prof = *P.by_index[u.ctx];
  UpdateCandidate out;
  out.context = prof.context;
  out.kind = u.kind == KVT_RECOMPRESS ? PlacementAction::Kind::Recompress : PlacementAction::Kind::Evict;
  out.target = candidate(prof, store.tiers(), u.tier_index, sp.names[u.method], u.ratio, u.size_bytes, u.quality,
                         u.ttft, u.utility);
  out.utility_drop = u.utility_drop;
  out.bytes_freed = u.bytes_freed;
  return out;
}

void resolve_overflow(StoreState& store, const ProfileMap& profiles, const CandidateSpace& space,
                      const UtilityParams& params, std::vector<PlacementAction>& actions) {
  const Space sp(space);
  const Profiles P(ordered(profiles), sp);
  Mirror mir(store, profiles, sp);
  const kvt_params pr{params.alpha};
  int64_t n = 0;
  const int rc = kvt_resolve_overflow(mir.s, P.p, &sp.s, &pr, &n);
  // the reference applies every step before it throws: replay what ran
  apply(store, mir.actions(n), P, sp, [](int32_t) { return std::pair<int64_t, int64_t>{0, 0}; }, actions);
  check(rc);
}

std::vector<PlacementAction> insert_joint(StoreState& store, const ContextId& context, const ProfileMap& profiles,
                                          const CandidateSpace& space, const UtilityParams& params,
                                          std::int64_t frequency, std::int64_t stamp, SelectionRule rule) {
  const Space sp(space);
  const Profiles P(ordered(profiles), sp);
  if (store.contains(context)) throw ValidationError("context " + context + " is already resident");
  const int32_t c = ctx_index(profiles, context);
  Mirror mir(store, profiles, sp);
  const kvt_params pr{params.alpha};
  int64_t n = 0, done = 0;
  const int rc = kvt_insert_joint(mir.s, P.p, &sp.s, &pr,
                                  rule == SelectionRule::QualityFirst ? KVT_RULE_QUALITY_FIRST : KVT_RULE_UTILITY,
                                  &c, &frequency, &stamp, 1, &n, &done);
  std::vector<PlacementAction> out;
  apply(store, mir.actions(n), P, sp, [&](int32_t) { return std::pair<int64_t, int64_t>{frequency, stamp}; }, out);
  check(rc);
  return out;
}

std::vector<PlacementAction> rearrange(StoreState& store, const ProfileMap& profiles, const CandidateSpace& space,
                                       const UtilityParams& params, SelectionRule rule) {
  const Space sp(space);
  const Profiles P(ordered(profiles), sp);
  Mirror mir(store, profiles, sp);
  // access stats survive the re-insert (placement.cpp:262-266)
  std::vector<std::pair<int64_t, int64_t>> stats(profiles.size(), {0, 0});
  for (size_t ti = 0; ti < store.tier_count(); ++ti)
    for (const CacheEntry& e : store.residents(ti))
      stats[static_cast<size_t>(ctx_index(profiles, e.context))] = {e.frequency, e.last_access};
  const kvt_params pr{params.alpha};
  int64_t n = 0;
  const int rc = kvt_rearrange(mir.s, P.p, &sp.s, &pr,
                               rule == SelectionRule::QualityFirst ? KVT_RULE_QUALITY_FIRST : KVT_RULE_UTILITY, &n);
  check(rc);
  store.clear();
  std::vector<PlacementAction> out;
  apply(store, mir.actions(n), P, sp, [&](int32_t c) { return stats[static_cast<size_t>(c)]; }, out);
  return out;
}

double placement_utility(const StoreState& store, const ProfileMap& profiles, const MethodSet& methods,
                         const UtilityParams& params) {
  const Space sp(methods, {1.0});
  const Profiles P(ordered(profiles), sp);
  Mirror mir(store, profiles, sp);
  const kvt_params pr{params.alpha};
  double total = 0.0;
  check(kvt_placement_utility(mir.s, P.p, &sp.s, &pr, &total));
  return total;
}

}  // namespace kvtier
