// TEST INFRASTRUCTURE ONLY. Exposes the UNMODIFIED reference library
// (kvtier, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/) through the ref_* copy of the C ABI in include/kvt_b200.h,
// so tests and bench.py's reference arm can drive it with the same arrays
// as the CUDA path. This file translates arrays <-> kvtier types and calls
// the reference's public API. One exception, clearly separated at the end:
// ref_insert_joint_cached, the single-core CPU baseline of the cached greedy
// built on the reference's own scoring functions, so the
// bench can separate the algorithmic speed-up from the hardware speed-up.
#include <cstdint>
#include <cstring>
#include <set>
#include <tuple>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "kvt_b200.h"
#include "kvtier/core.hpp"
#include "kvtier/placement.hpp"
#include "kvtier/quality.hpp"
#include "kvtier/utility.hpp"

extern "C" {
KVT_DECLARE_API(ref_)
}

namespace {

thread_local std::string g_err;

// Context index <-> ContextId: zero padded so byte order == index order.
std::string ctx_name(int32_t c) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "c%09d", c);
  return buf;
}
int32_t ctx_index(const std::string& id) { return std::stoi(id.substr(1)); }

template <class F>
int guard(F&& f) {
  try {
    f();
    return KVT_OK;
  } catch (const kvtier::ValidationError& e) {
    g_err = e.what();
    return KVT_EVALIDATION;
  } catch (const kvtier::TraceError& e) {
    g_err = e.what();
    return KVT_ETRACE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KVT_EINVAL;
  }
}

kvtier::CandidateSpace make_space(const kvt_space* sp) {
  std::vector<kvtier::CompressionMethod> ms;
  for (int m = 0; m < sp->n_methods; ++m)
    ms.push_back({sp->method_names[m], sp->decompression_overhead[m]});
  std::vector<double> rs(sp->ratios, sp->ratios + sp->n_ratios);
  return kvtier::CandidateSpace(kvtier::MethodSet(std::move(ms)), std::move(rs));
}

std::vector<kvtier::TierSpec> make_tiers(const kvt_tier* t, int32_t n) {
  std::vector<kvtier::TierSpec> out;
  for (int i = 0; i < n; ++i) {
    kvtier::TierSpec s;
    s.tier_id = t[i].tier_id;
    s.name = "t" + std::to_string(t[i].tier_id);
    if (!t[i].unlimited) s.capacity_bytes = t[i].capacity_bytes;
    s.read_bandwidth = t[i].read_bandwidth;
    s.fixed_access_latency = t[i].fixed_access_latency;
    out.push_back(s);
  }
  return out;
}

int method_index(const kvtier::CandidateSpace& space, const std::string& name) {
  const auto& ms = space.methods().methods();
  for (size_t i = 0; i < ms.size(); ++i)
    if (ms[i].name == name) return static_cast<int>(i);
  return -1;
}

}  // namespace

struct kvt_handle {
  int unused = 0;
};

struct kvt_pset {
  kvt_profiles raw{};
  std::vector<int64_t> orig;
  std::vector<double> freq, grid, qual;
  std::vector<int32_t> goff;
  std::vector<uint8_t> has;
  // ProfileMap built against one method-name list (cached by names).
  std::vector<std::string> names;
  kvtier::ProfileMap map;

  const kvtier::ProfileMap& profiles(const kvt_space* sp) {
    std::vector<std::string> want(sp->method_names, sp->method_names + sp->n_methods);
    if (want == names && !map.empty()) return map;
    names = want;
    map.clear();
    const int M = raw.n_methods;
    for (int32_t c = 0; c < raw.n_ctx; ++c) {
      kvtier::ContextProfile p;
      p.context = ctx_name(c);
      p.original_size_bytes = orig[c];
      p.frequency = freq[c];
      const int32_t g0 = goff[c], len = goff[c + 1] - g0;
      p.ratio_grid.assign(grid.begin() + g0, grid.begin() + g0 + len);
      for (int m = 0; m < M; ++m) {
        if (!has[static_cast<size_t>(c) * M + m]) continue;
        const double* row = qual.data() + static_cast<size_t>(g0) * M + static_cast<size_t>(m) * len;
        p.quality_table[names[m]] = std::vector<double>(row, row + len);
      }
      map.emplace(p.context, std::move(p));
    }
    return map;
  }
};

struct kvt_store {
  std::unique_ptr<kvtier::StoreState> st;
  int32_t n_ctx = 0;
  std::vector<kvt_action> act;
  std::vector<std::string> names;  // method names of the last space seen
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_abi_version(void) { return KVT_ABI_VERSION; }

int ref_create(int, void*, kvt_handle** out) {
  *out = new kvt_handle();
  return KVT_OK;
}
int ref_destroy(kvt_handle* h) {
  delete h;
  return KVT_OK;
}

int ref_pset_create(kvt_handle*, const kvt_profiles* pr, kvt_pset** out) {
  auto* p = new kvt_pset();
  const int32_t n = pr->n_ctx, M = pr->n_methods, G = pr->grid_offset[n];
  p->raw = *pr;
  p->orig.assign(pr->original_size_bytes, pr->original_size_bytes + n);
  p->freq.assign(pr->frequency, pr->frequency + n);
  p->goff.assign(pr->grid_offset, pr->grid_offset + n + 1);
  p->grid.assign(pr->grid, pr->grid + G);
  p->qual.assign(pr->quality, pr->quality + static_cast<size_t>(G) * M);
  p->has.assign(pr->has_method, pr->has_method + static_cast<size_t>(n) * M);
  *out = p;
  return KVT_OK;
}
int ref_pset_destroy(kvt_pset* p) {
  delete p;
  return KVT_OK;
}

int ref_score_candidates(kvt_handle*, const kvt_pset* pc, const kvt_tier* tiers, int32_t n_tiers,
                         const kvt_space* sp, const kvt_params* params, int64_t* size,
                         double* quality, uint8_t* valid, double* ttft, double* utility) {
  auto* p = const_cast<kvt_pset*>(pc);
  return guard([&] {
    const auto space = make_space(sp);
    const auto hier = kvtier::validate_hierarchy(make_tiers(tiers, n_tiers));
    const auto& map = p->profiles(sp);
    kvtier::UtilityParams up;
    up.alpha = params->alpha;
    const int T = static_cast<int>(hier.size()), M = sp->n_methods;
    const int R = static_cast<int>(space.ratios().size());
    int32_t c = 0;
    for (const auto& [id, prof] : map) {
      if (size)
        for (int r = 0; r < R; ++r)
          size[static_cast<size_t>(c) * R + r] =
              kvtier::compressed_size(prof.original_size_bytes, space.ratios()[r]);
      if (valid) std::memset(valid + static_cast<size_t>(c) * M * R, 0, static_cast<size_t>(M) * R);
      if (quality)
        for (int k = 0; k < M * R; ++k) quality[static_cast<size_t>(c) * M * R + k] = 0.0;
      for (int k = 0; k < T * M * R; ++k) {
        if (ttft) ttft[static_cast<size_t>(c) * T * M * R + k] = 0.0;
        if (utility) utility[static_cast<size_t>(c) * T * M * R + k] = 0.0;
      }
      for (const auto& cand : kvtier::all_candidates(prof, hier, space, up)) {
        const int m = method_index(space, cand.config.method);
        int r = 0;
        while (space.ratios()[r] != cand.config.ratio) ++r;
        const size_t qi = (static_cast<size_t>(c) * M + m) * R + r;
        const size_t ui = ((static_cast<size_t>(c) * T + cand.tier_index) * M + m) * R + r;
        if (valid) valid[qi] = 1;
        if (quality) quality[qi] = cand.quality;
        if (ttft) ttft[ui] = cand.ttft;
        if (utility) utility[ui] = cand.utility;
      }
      ++c;
    }
  });
}

int ref_best_config(kvt_handle*, const kvt_pset* pc, const kvt_tier* tiers, int32_t n_tiers,
                    const kvt_space* sp, const kvt_params* params, int32_t rule, kvt_best* out) {
  auto* p = const_cast<kvt_pset*>(pc);
  return guard([&] {
    const auto space = make_space(sp);
    const auto hier = kvtier::validate_hierarchy(make_tiers(tiers, n_tiers));
    const auto& map = p->profiles(sp);
    kvtier::UtilityParams up;
    up.alpha = params->alpha;
    int32_t c = 0;
    for (const auto& [id, prof] : map) {
      kvt_best& b = out[c++];
      std::memset(&b, 0, sizeof b);
      try {
        const auto best = kvtier::best_config(
            prof, hier, space, up,
            rule == KVT_RULE_QUALITY_FIRST ? kvtier::SelectionRule::QualityFirst
                                           : kvtier::SelectionRule::Utility);
        b.tier_index = best.tier_index;
        b.tier_id = best.tier_id;
        b.method = method_index(space, best.config.method);
        int r = 0;
        while (space.ratios()[r] != best.config.ratio) ++r;
        b.ratio_index = r;
        b.ratio = best.config.ratio;
        b.size_bytes = best.size_bytes;
        b.quality = best.quality;
        b.ttft = best.ttft;
        b.utility = best.utility;
      } catch (const kvtier::ValidationError&) {
        b.status = 1;
      }
    }
  });
}

int ref_oracle_mckp(kvt_handle*, const kvt_pset* pc, const kvt_tier* tiers, int32_t n_tiers,
                    const kvt_space* sp, const kvt_params* params, double max_assignments,
                    double* total_utility, kvt_best* out) {
  auto* p = const_cast<kvt_pset*>(pc);
  return guard([&] {
    const auto space = make_space(sp);
    const auto& map = p->profiles(sp);
    std::vector<kvtier::ContextProfile> profs;
    for (const auto& [id, prof] : map) profs.push_back(prof);
    kvtier::UtilityParams up;
    up.alpha = params->alpha;
    const auto res = kvtier::oracle_mckp(profs, make_tiers(tiers, n_tiers), space, up, max_assignments);
    *total_utility = res.total_utility;
    int32_t c = 0;
    for (const auto& [id, prof] : map) {
      const auto& best = res.assignment.at(id);
      kvt_best& b = out[c++];
      std::memset(&b, 0, sizeof b);
      b.tier_index = best.tier_index;
      b.tier_id = best.tier_id;
      b.method = method_index(space, best.config.method);
      int r = 0;
      while (space.ratios()[r] != best.config.ratio) ++r;
      b.ratio_index = r;
      b.ratio = best.config.ratio;
      b.size_bytes = best.size_bytes;
      b.quality = best.quality;
      b.ttft = best.ttft;
      b.utility = best.utility;
    }
  });
}

int ref_store_create(kvt_handle*, const kvt_tier* tiers, int32_t n_tiers, int32_t n_ctx,
                     kvt_store** out) {
  return guard([&] {
    auto* s = new kvt_store();
    s->st = std::make_unique<kvtier::StoreState>(make_tiers(tiers, n_tiers));
    s->n_ctx = n_ctx;
    *out = s;
  });
}
int ref_store_destroy(kvt_store* s) {
  delete s;
  return KVT_OK;
}

namespace {
std::string method_name_for(const kvt_store* s, int32_t m) {
  if (m >= 0 && m < static_cast<int32_t>(s->names.size())) return s->names[m];
  return "m" + std::to_string(m);
}
}  // namespace

int ref_store_add(kvt_store* s, int32_t ctx, const kvt_entry* e) {
  return guard([&] {
    kvtier::CacheEntry ce;
    ce.context = ctx_name(ctx);
    ce.original_size_bytes = e->original_size_bytes;
    ce.config = {method_name_for(s, e->method), e->ratio};
    if (e->tier_index < 0 || e->tier_index >= static_cast<int>(s->st->tier_count()))
      throw kvtier::ValidationError("unknown tier index");
    ce.tier = s->st->tier(e->tier_index).tier_id;
    ce.frequency = e->frequency;
    ce.last_access = e->last_access;
    s->st->add(ce);
  });
}

int ref_store_remove(kvt_store* s, int32_t ctx, kvt_entry* removed) {
  return guard([&] {
    const size_t ti = s->st->tier_index_of(ctx_name(ctx));
    const auto e = s->st->remove(ctx_name(ctx));
    if (removed) {
      removed->tier_index = static_cast<int32_t>(ti);
      removed->ratio = e.config.ratio;
      removed->original_size_bytes = e.original_size_bytes;
      removed->frequency = e.frequency;
      removed->last_access = e.last_access;
      removed->method = 0;
      for (size_t m = 0; m < s->names.size(); ++m)
        if (s->names[m] == e.config.method) removed->method = static_cast<int32_t>(m);
      removed->seq = 0;
    }
  });
}

int ref_store_reconfigure(kvt_store* s, int32_t ctx, int32_t m, double ratio) {
  return guard([&] { s->st->reconfigure(ctx_name(ctx), {method_name_for(s, m), ratio}); });
}
int ref_store_touch(kvt_store* s, int32_t ctx, int64_t stamp) {
  return guard([&] { s->st->touch(ctx_name(ctx), stamp); });
}
int ref_store_touch_many(kvt_store* s, const int32_t* ctx, const int64_t* stamps, int64_t n) {
  return guard([&] {
    for (int64_t i = 0; i < n; ++i) s->st->touch(ctx_name(ctx[i]), stamps[i]);
  });
}
int ref_store_clear(kvt_store* s) {
  s->st->clear();
  return KVT_OK;
}
int ref_store_occupancy(kvt_store* s, int64_t* occ) {
  for (size_t t = 0; t < s->st->tier_count(); ++t) occ[t] = s->st->occupancy(t);
  return KVT_OK;
}

int ref_store_snapshot(kvt_store* s, kvt_entry* out) {
  for (int32_t c = 0; c < s->n_ctx; ++c) {
    std::memset(&out[c], 0, sizeof(kvt_entry));
    out[c].tier_index = -1;
  }
  int64_t seq = 0;
  for (size_t t = 0; t < s->st->tier_count(); ++t) {
    for (const auto& e : s->st->residents(t)) {
      const int32_t c = ctx_index(e.context);
      kvt_entry& o = out[c];
      o.tier_index = static_cast<int32_t>(t);
      o.method = -1;
      for (size_t m = 0; m < s->names.size(); ++m)
        if (s->names[m] == e.config.method) o.method = static_cast<int32_t>(m);
      o.ratio = e.config.ratio;
      o.original_size_bytes = e.original_size_bytes;
      o.frequency = e.frequency;
      o.last_access = e.last_access;
      o.seq = seq++;  // position order within the tier (arrival order)
    }
  }
  return KVT_OK;
}

int ref_store_actions(kvt_store* s, kvt_action* out, int64_t n) {
  if (n > static_cast<int64_t>(s->act.size())) n = static_cast<int64_t>(s->act.size());
  std::memcpy(out, s->act.data(), sizeof(kvt_action) * static_cast<size_t>(n));
  return KVT_OK;
}

namespace {
void set_names(kvt_store* s, const kvt_space* sp) {
  s->names.assign(sp->method_names, sp->method_names + sp->n_methods);
}
void append(kvt_store* s, const kvtier::CandidateSpace& space,
            const std::vector<kvtier::PlacementAction>& acts) {
  for (const auto& a : acts) {
    kvt_action o;
    o.kind = a.kind == kvtier::PlacementAction::Kind::Insert       ? KVT_INSERT
             : a.kind == kvtier::PlacementAction::Kind::Recompress ? KVT_RECOMPRESS
                                                                   : KVT_EVICT;
    o.ctx = ctx_index(a.context);
    o.tier_id = a.tier;
    o.method = method_index(space, a.config.method);
    o.ratio = a.config.ratio;
    s->act.push_back(o);
  }
}
kvtier::UtilityParams mk_params(const kvt_params* p) {
  kvtier::UtilityParams up;
  up.alpha = p->alpha;
  return up;
}
}  // namespace

int ref_least_drop_update(kvt_store* s, const kvt_pset* pc, const kvt_space* sp,
                          const kvt_params* params, int32_t tier_index, kvt_update* out) {
  auto* p = const_cast<kvt_pset*>(pc);
  set_names(s, sp);
  return guard([&] {
    const auto space = make_space(sp);
    const auto u = kvtier::least_drop_update(*s->st, static_cast<size_t>(tier_index),
                                             p->profiles(sp), space, mk_params(params));
    out->ctx = ctx_index(u.context);
    out->kind = u.kind == kvtier::PlacementAction::Kind::Recompress ? KVT_RECOMPRESS : KVT_EVICT;
    out->tier_index = u.target.tier_index;
    out->tier_id = u.target.tier_id;
    out->method = method_index(space, u.target.config.method);
    out->pad_ = 0;
    out->ratio = u.target.config.ratio;
    out->size_bytes = u.target.size_bytes;
    out->quality = u.target.quality;
    out->ttft = u.target.ttft;
    out->utility = u.target.utility;
    out->utility_drop = u.utility_drop;
    out->bytes_freed = u.bytes_freed;
  });
}

int ref_resolve_overflow(kvt_store* s, const kvt_pset* pc, const kvt_space* sp,
                         const kvt_params* params, int64_t* n_actions) {
  auto* p = const_cast<kvt_pset*>(pc);
  set_names(s, sp);
  s->act.clear();
  int rc = guard([&] {
    const auto space = make_space(sp);
    std::vector<kvtier::PlacementAction> acts;
    try {
      kvtier::resolve_overflow(*s->st, p->profiles(sp), space, mk_params(params), acts);
    } catch (...) {
      append(s, space, acts);
      throw;
    }
    append(s, space, acts);
  });
  *n_actions = static_cast<int64_t>(s->act.size());
  return rc;
}

int ref_insert_joint(kvt_store* s, const kvt_pset* pc, const kvt_space* sp,
                     const kvt_params* params, int32_t rule, const int32_t* ctx,
                     const int64_t* frequency, const int64_t* stamp, int64_t n_ops,
                     int64_t* n_actions, int64_t* n_done) {
  auto* p = const_cast<kvt_pset*>(pc);
  set_names(s, sp);
  s->act.clear();
  *n_done = 0;
  int rc = guard([&] {
    const auto space = make_space(sp);
    const auto& map = p->profiles(sp);
    const auto up = mk_params(params);
    const auto sel = rule == KVT_RULE_QUALITY_FIRST ? kvtier::SelectionRule::QualityFirst
                                                    : kvtier::SelectionRule::Utility;
    for (int64_t i = 0; i < n_ops; ++i) {
      const auto acts = kvtier::insert_joint(*s->st, ctx_name(ctx[i]), map, space, up,
                                             frequency ? frequency[i] : 0, stamp ? stamp[i] : 0, sel);
      append(s, space, acts);
      *n_done = i + 1;
    }
  });
  *n_actions = static_cast<int64_t>(s->act.size());
  return rc;
}

int ref_rearrange(kvt_store* s, const kvt_pset* pc, const kvt_space* sp, const kvt_params* params,
                  int32_t rule, int64_t* n_actions) {
  auto* p = const_cast<kvt_pset*>(pc);
  set_names(s, sp);
  s->act.clear();
  int rc = guard([&] {
    const auto space = make_space(sp);
    const auto acts = kvtier::rearrange(
        *s->st, p->profiles(sp), space, mk_params(params),
        rule == KVT_RULE_QUALITY_FIRST ? kvtier::SelectionRule::QualityFirst
                                       : kvtier::SelectionRule::Utility);
    append(s, space, acts);
  });
  *n_actions = static_cast<int64_t>(s->act.size());
  return rc;
}

int ref_placement_utility(kvt_store* s, const kvt_pset* pc, const kvt_space* sp,
                          const kvt_params* params, double* out) {
  auto* p = const_cast<kvt_pset*>(pc);
  set_names(s, sp);
  return guard([&] {
    const auto space = make_space(sp);
    *out = kvtier::placement_utility(*s->st, p->profiles(sp), space.methods(), mk_params(params));
  });
}

}  // extern "C"

extern "C" int ref_store_bind_space(kvt_store* s, const kvt_space* sp) {
  set_names(s, sp);
  return KVT_OK;
}

// ---------------------------------------------------------------------------
// Serve-loop goldens: load a reference scenario file with the
// reference's own loader, run the reference's own replay, and write the
// expanded scenario (every input the replay used) plus its results as JSON.
// Test infrastructure only: tests/golden/make_replay_golden.py calls it here
// (the container with /root/reference), the fixtures travel, the GPU box
// never runs this.
#include <fstream>

#include "kvtier/simulate.hpp"
#include "kvtier/workload.hpp"
#include "json.hpp"  // nlohmann/json 3.11.3, the reference build's copy (oracle/Makefile NLOHMANN)

extern "C" int ref_replay_dump(const char* scenario_path, const char* out_path, const char* const* overrides,
                               int32_t n_overrides) {
  return guard([&] {
    using nlohmann::json;
    std::vector<std::string> ov;
    for (int32_t i = 0; i < n_overrides; ++i) ov.emplace_back(overrides[i]);
    const kvtier::LoadedScenario run = kvtier::load_scenario_file(scenario_path, ov);
    const kvtier::Scenario& sc = run.scenario;
    json j;
    j["policy"] = run.policy.label();
    j["policy_kind"] = static_cast<int>(run.policy.kind);
    j["rule"] = run.policy.rule == kvtier::SelectionRule::Utility ? "utility" : "quality_first";
    j["warm_start"] = sc.warm_start;
    j["miss_store_bottom"] = sc.miss_store_bottom;
    j["drift"] = sc.drift.enabled;
    j["seed"] = sc.seed;
    j["drift_config"] = {{"threshold", sc.drift.threshold},
                         {"min_samples", sc.drift.min_samples},
                         {"window_size", sc.drift.window_size},
                         {"gpu_window", sc.drift.gpu_window},
                         {"max_batch", sc.drift.max_batch},
                         {"duration", sc.drift.reprofile.duration},
                         {"penalty", sc.drift.reprofile.penalty},
                         {"noise_amplitude", sc.drift.reprofile.noise_amplitude}};
    j["n_truth"] = sc.truth.size();
    j["params"] = {{"alpha", sc.params.alpha}, {"prefill_a", sc.params.prefill_a},
                   {"prefill_b", sc.params.prefill_b}, {"bytes_per_token", sc.params.bytes_per_token}};
    for (const auto& t : sc.tiers) {
      json jt = {{"tier_id", t.tier_id}, {"name", t.name}, {"read_bandwidth", t.read_bandwidth},
                 {"fixed_access_latency", t.fixed_access_latency}};
      jt["capacity_bytes"] = t.capacity_bytes ? json(*t.capacity_bytes) : json(nullptr);
      j["tiers"].push_back(jt);
    }
    for (const auto& m : sc.space.methods().methods())
      j["methods"].push_back({{"name", m.name}, {"decompression_overhead", m.decompression_overhead}});
    j["ratios"] = sc.space.ratios();
    for (const auto& [id, p] : sc.profiles) {
      json jp = {{"context", id}, {"size", p.original_size_bytes}, {"frequency", p.frequency},
                 {"grid", p.ratio_grid}};
      for (const auto& [m, q] : p.quality_table) jp["quality"][m] = q;
      j["profiles"].push_back(jp);
    }
    for (const auto& [id, curve] : sc.truth)
      for (const auto& [m, sc_] : curve.per_method) j["truth"][id][m] = {sc_.sensitivity, sc_.shape_k};
    j["order"] = sc.order;
    for (const auto& r : run.trace)
      j["trace"].push_back({{"t", r.t}, {"context", r.context}, {"n_new_tokens", r.n_new_tokens}});
    const kvtier::ReplayResult res = kvtier::replay(run.trace, run.policy, sc);
    json jr;
    for (const auto& r : res.records)
      jr["records"].push_back({{"hit", r.outcome == kvtier::Outcome::Hit}, {"tier", r.tier},
                               {"method", r.config.method}, {"ratio", r.config.ratio}, {"ttft", r.ttft},
                               {"quality", r.quality}});
    for (const auto& a : res.actions)
      jr["actions"].push_back({{"kind", kvtier::to_string(a.kind)}, {"context", a.context}, {"tier", a.tier},
                               {"method", a.config.method}, {"ratio", a.config.ratio}});
    jr["final_placements"] = res.final_placements;
    const auto& m = res.metrics;
    jr["metrics"] = {{"n_requests", m.n_requests}, {"sum_ttft", m.sum_ttft}, {"mean_ttft", m.mean_ttft},
                     {"p50_ttft", m.p50_ttft}, {"p90_ttft", m.p90_ttft}, {"p99_ttft", m.p99_ttft},
                     {"mean_quality", m.mean_quality}, {"miss_fraction", m.miss_fraction}};
    for (const auto& [tier, f] : m.hit_fraction_by_tier) jr["metrics"]["hit_fraction_by_tier"][std::to_string(tier)] = f;
    jr["reprofile_count"] = res.reprofile_count;
    for (const auto& w : res.profiling_windows)
      jr["profiling_windows"].push_back({{"start", w.start}, {"duration", w.duration}, {"penalty", w.penalty}});
    j["result"] = jr;
    std::ofstream(out_path) << j.dump(1);
  });
}

// ------------------------------------------------------------------------
// CPU BASELINE (not the reference's algorithm, not the product): insert_joint
// (proj/src/placement.cpp:225-250) with least_drop_update's rescan of every
// resident (:174-204) replaced by a cached per-resident best update and one
// ordered set per tier keyed (utility_drop, -bytes_freed, context) — the
// structure SURVEY.md §0.6 validated as bit-identical, and the one the
// device greedy (K3) implements. A resident's options depend only on its own
// entry and profile (enumerate_updates, proj/src/utility.cpp:81-127), so only
// the resident a step changes (or a new insert) is re-scored. Uses the
// reference's StoreState, best_config, score_candidate and enumerate_updates.
namespace {
struct CachedBest {
  bool valid = false;
  kvtier::UpdateCandidate u;
};
using Key = std::tuple<double, int64_t, std::string>;  // (drop, -bytes_freed, context)

bool better_option(const kvtier::UpdateCandidate& a, const kvtier::UpdateCandidate& b) {
  if (a.utility_drop != b.utility_drop) return a.utility_drop < b.utility_drop;
  return a.bytes_freed > b.bytes_freed;  // same resident: first enumerated wins the rest
}

CachedBest resident_best(const kvtier::StoreState& st, const kvtier::CacheEntry& e, size_t ti,
                         const kvtier::ContextProfile& prof, const kvtier::CandidateSpace& space,
                         const kvtier::UtilityParams& up) {
  CachedBest b;
  const kvtier::ConfigCandidate cur =
      kvtier::score_candidate(prof, e.config, st.tier(ti), static_cast<int>(ti), space.methods(), up);
  for (const auto& opt : kvtier::enumerate_updates(e, prof, st.tiers(), space, up)) {
    kvtier::UpdateCandidate u;
    u.context = e.context;
    u.kind = opt.tier_index == static_cast<int>(ti) ? kvtier::PlacementAction::Kind::Recompress
                                                    : kvtier::PlacementAction::Kind::Evict;
    u.target = opt;
    u.utility_drop = cur.utility - opt.utility;
    u.bytes_freed = u.kind == kvtier::PlacementAction::Kind::Recompress ? cur.size_bytes - opt.size_bytes
                                                                       : cur.size_bytes;
    if (!b.valid || better_option(u, b.u)) {
      b.u = u;
      b.valid = true;
    }
  }
  return b;
}
}  // namespace

extern "C" int ref_insert_joint_cached(kvt_store* s, const kvt_pset* pc, const kvt_space* sp,
                                       const kvt_params* params, int32_t rule, const int32_t* ctx,
                                       const int64_t* frequency, const int64_t* stamp, int64_t n_ops,
                                       int64_t* n_actions, int64_t* n_done) {
  auto* p = const_cast<kvt_pset*>(pc);
  set_names(s, sp);
  s->act.clear();
  *n_done = 0;
  int rc = guard([&] {
    const auto space = make_space(sp);
    const auto& map = p->profiles(sp);
    const auto up = mk_params(params);
    const auto sel = rule == KVT_RULE_QUALITY_FIRST ? kvtier::SelectionRule::QualityFirst
                                                    : kvtier::SelectionRule::Utility;
    kvtier::StoreState& st = *s->st;
    const size_t T = st.tier_count();
    std::vector<std::set<Key>> sets(T);
    std::map<std::string, CachedBest> cache;
    auto key_of = [](const kvtier::UpdateCandidate& u) { return Key(u.utility_drop, -u.bytes_freed, u.context); };
    auto enter = [&](const kvtier::CacheEntry& e, size_t ti) {
      CachedBest b = resident_best(st, e, ti, map.at(e.context), space, up);
      if (b.valid) sets[ti].insert(key_of(b.u));
      cache[e.context] = std::move(b);
    };
    auto leave = [&](const std::string& c, size_t ti) {
      auto it = cache.find(c);
      if (it != cache.end() && it->second.valid) sets[ti].erase(key_of(it->second.u));
    };
    for (size_t ti = 0; ti < T; ++ti)
      for (const auto& e : st.residents(ti)) enter(e, ti);
    for (int64_t i = 0; i < n_ops; ++i) {
      const std::string id = ctx_name(ctx[i]);
      if (st.contains(id)) throw kvtier::ValidationError("context " + id + " is already resident");
      const kvtier::ContextProfile& prof = map.at(id);
      const kvtier::ConfigCandidate best = kvtier::best_config(prof, st.tiers(), space, up, sel);
      kvtier::CacheEntry entry;
      entry.context = id;
      entry.original_size_bytes = prof.original_size_bytes;
      entry.config = best.config;
      entry.tier = best.tier_id;
      entry.frequency = frequency ? frequency[i] : 0;
      entry.last_access = stamp ? stamp[i] : 0;
      st.add(entry);
      std::vector<kvtier::PlacementAction> acts{{kvtier::PlacementAction::Kind::Insert, id, best.tier_id, best.config}};
      enter(*st.find(id), st.tier_index_of(id));
      while (auto over = st.first_over_capacity()) {
        if (sets[*over].empty())
          throw kvtier::ValidationError("tier " + st.tier(*over).name +
                                        " is over capacity and no resident has a space-saving option");
        const std::string who = std::get<2>(*sets[*over].begin());
        const kvtier::UpdateCandidate u = cache.at(who).u;
        leave(who, *over);
        if (u.kind == kvtier::PlacementAction::Kind::Recompress) {
          st.reconfigure(u.context, u.target.config);
        } else {
          kvtier::CacheEntry moved = st.remove(u.context);
          moved.tier = u.target.tier_id;
          moved.config = u.target.config;
          st.add(std::move(moved));
        }
        enter(*st.find(who), st.tier_index_of(who));
        acts.push_back({u.kind, u.context, u.target.tier_id, u.target.config});
      }
      append(s, space, acts);
      *n_done = i + 1;
    }
  });
  *n_actions = static_cast<int64_t>(s->act.size());
  return rc;
}
