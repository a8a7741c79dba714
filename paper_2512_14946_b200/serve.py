"""Cache-manager serve loop around the device store.

Host mirror of `kvtier::Replayer` (proj/src/simulate.cpp:63-86, 130-227,
246-251) for the joint policy: a trace of (t, context, n_new_tokens)
requests against the placement kept in a `StoreState` (the CUDA store of
`libkvt_b200.so`). Placement only changes on a miss, so the loop runs in
segments: every hit up to the next miss is served from a host copy of the
placement (tier, method, ratio per context) with the reference's TTFT /
quality arithmetic, the segment's touches go to the device store in one
`store_touch_many`, and the miss runs `insert_joint` (K1 scoring + the K3
greedy) on the device, after which the host copy is refreshed from one
snapshot. Records, actions, final placements and metrics come out in the
reference's `ReplayResult` shape.

Not here yet (SURVEY §8 f3 and the baselines): drift tracking and
re-profiling, `miss_store_bottom`, and the LRU / fixed / impress /
prefill policies; `Replayer` refuses scenarios that need them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A
from .kvtier import (CandidateSpace, CompressionMethod, ContextProfile, Engine, ProfileArrays, TierSpec,
                     UtilityParams, sorted_tiers)

KIND_NAMES = {A.KVT_INSERT: "insert", A.KVT_RECOMPRESS: "recompress", A.KVT_EVICT: "evict"}
GRID_EPS = 1e-9  # kGridEps, proj/src/quality.cpp


@dataclass
class Request:  # proj/include/kvtier/simulate.hpp:22-26
    t: float
    context: str
    n_new_tokens: int = 0


@dataclass
class RequestRecord:  # proj/include/kvtier/simulate.hpp:31-38
    request: Request
    hit: bool = False
    tier: int = -1  # serving tier id on a hit
    method: str = ""
    ratio: float = 1.0
    ttft: float = 0.0
    quality: float = 1.0


@dataclass
class ReplayResult:  # proj/include/kvtier/simulate.hpp:82-90
    records: List[RequestRecord]
    metrics: Dict[str, object]
    final_placements: Dict[str, int]
    actions: List[Tuple[str, str, int, str, float]]  # (kind, context, tier id, method, ratio)


@dataclass
class Scenario:
    """Everything a replay needs besides the trace (simulate.hpp:65-76), in
    expanded form: tiers, params, space, profiles and truth curves as data."""
    tiers: List[TierSpec]
    params: UtilityParams
    space: CandidateSpace
    profiles: List[ContextProfile]
    truth: Dict[str, Dict[str, Tuple[float, float]]] = field(default_factory=dict)  # ctx -> method -> (s, k)
    order: List[str] = field(default_factory=list)
    warm_start: bool = False
    miss_store_bottom: bool = False
    drift: bool = False
    rule: str = "utility"

    @staticmethod
    def from_doc(doc: dict) -> Tuple["Scenario", List[Request]]:
        """The expanded scenario JSON (tests/golden/make_replay_golden.py)."""
        tiers = [TierSpec(int(t["tier_id"]), t.get("name", ""), t["capacity_bytes"], float(t["read_bandwidth"]),
                          float(t["fixed_access_latency"])) for t in doc["tiers"]]
        p = doc["params"]
        params = UtilityParams(float(p["alpha"]), float(p["prefill_a"]), float(p["prefill_b"]),
                               float(p["bytes_per_token"]))
        space = CandidateSpace([CompressionMethod(m["name"], float(m["decompression_overhead"]))
                                for m in doc["methods"]], [float(r) for r in doc["ratios"]])
        profiles = [ContextProfile(q["context"], int(q["size"]), float(q["frequency"]),
                                   [float(x) for x in q["grid"]],
                                   {m: [float(x) for x in v] for m, v in q.get("quality", {}).items()})
                    for q in doc["profiles"]]
        truth = {c: {m: (float(v[0]), float(v[1])) for m, v in per.items()}
                 for c, per in (doc.get("truth") or {}).items()}
        sc = Scenario(tiers, params, space, profiles, truth, list(doc.get("order") or []),
                      bool(doc.get("warm_start")), bool(doc.get("miss_store_bottom")), bool(doc.get("drift")),
                      doc.get("rule", "utility"))
        trace = [Request(float(r["t"]), r["context"], int(r.get("n_new_tokens", 0))) for r in doc["trace"]]
        return sc, trace


# --- the reference's serving arithmetic (host doubles, same operation order)

def compressed_size(orig: int, ratio: float) -> int:  # proj/src/core.cpp:72-84
    return max(1, int(math.floor(float(orig) * ratio + 0.5)))


def prefill_time(n_tokens: int, p: UtilityParams) -> float:  # proj/src/utility.cpp:43-49
    n = float(n_tokens)
    return p.prefill_a * n + p.prefill_b * n * n


def load_time(size: int, tier: TierSpec, ovh: float) -> float:  # proj/src/utility.cpp:51-59
    s = float(size)
    return tier.fixed_access_latency + s / tier.read_bandwidth + s * ovh


def token_count(orig: int, p: UtilityParams) -> int:  # proj/src/quality.cpp:28-31
    return max(1, int(math.floor(float(orig) / p.bytes_per_token + 0.5)))


def quality_of(prof: ContextProfile, method: str, ratio: float) -> float:  # proj/src/quality.cpp:86-113
    grid, values = prof.ratio_grid, prof.quality_table[method]
    key = ratio - GRID_EPS
    i = 0
    while i < len(grid) and grid[i] < key:  # std::lower_bound
        i += 1
    i = min(i, len(grid) - 1)
    if abs(grid[i] - ratio) <= GRID_EPS or i == 0:
        return values[i]
    x0, x1, y0, y1 = grid[i - 1], grid[i], values[i - 1], values[i]
    t = (ratio - x0) / (x1 - x0)
    return y0 + t * (y1 - y0)


def synth_quality(sensitivity: float, shape_k: float, ratio: float) -> float:  # proj/src/quality.cpp:115-127
    drop = sensitivity * math.pow((1.0 - ratio) / 0.1, shape_k)
    return min(max(1.0 - drop, 0.0), 1.0)


class Replayer:
    """kvtier::Replayer (joint policy) on the device store."""

    def __init__(self, eng: Engine, scenario: Scenario):
        if scenario.drift:
            raise NotImplementedError("drift / re-profiling (SURVEY §8 f3) is not in the serve loop yet")
        if scenario.miss_store_bottom:
            raise NotImplementedError("miss_store_bottom is not in the serve loop yet")
        self.sc = scenario
        self.eng = eng
        self.tiers = sorted_tiers(scenario.tiers)  # Replayer keeps the validated order
        self.arrays = ProfileArrays.from_profiles(scenario.profiles, scenario.space)
        self.prof = {p.context: p for p in scenario.profiles}
        self.ps = eng.pset(self.arrays)
        self.store = eng.store(self.tiers, self.arrays.n, scenario.space)
        self.rule = A.KVT_RULE_UTILITY if scenario.rule == "utility" else A.KVT_RULE_QUALITY_FIRST
        self.names = scenario.space.method_names
        self.ovh = [m.decompression_overhead for m in scenario.space.methods]
        self.stamp = 0
        self.actions: List[Tuple[str, str, int, str, float]] = []
        self.records: List[RequestRecord] = []
        self.last_t: Optional[float] = None
        self.n_device_calls = 0
        if scenario.warm_start:
            self._warm_up()
        self._refresh()

    # -- device store
    def _insert(self, ctx: Sequence[int], freq: Sequence[int], stamps: Sequence[int]):
        acts = self.store.insert_joint(self.ps, self.sc.space, self.sc.params, np.asarray(ctx, np.int32),
                                       frequency=np.asarray(freq, np.int64), stamp=np.asarray(stamps, np.int64),
                                       rule=self.rule)
        self.n_device_calls += 1
        ids = self.arrays.ids
        for a in acts:
            self.actions.append((KIND_NAMES[int(a["kind"])], ids[int(a["ctx"])], int(a["tier_id"]),
                                 self.names[int(a["method"])], float(a["ratio"])))

    def _refresh(self):
        snap = self.store.snapshot()
        self.tier_index = snap["tier_index"].astype(np.int64)
        self.method = snap["method"].astype(np.int64)
        self.ratio = snap["ratio"].astype(np.float64)
        self.seq = snap["seq"].astype(np.int64)

    def _warm_up(self):  # simulate.cpp:72-85: every context, frequency 0, one stamp each
        order = self.sc.order or sorted(self.prof, key=lambda c: c.encode())
        ctx = [self.arrays.index[c] for c in order]
        stamps = list(range(self.stamp, self.stamp + len(ctx)))
        self.stamp += len(ctx)
        self._insert(ctx, [0] * len(ctx), stamps)

    # -- serving
    def run(self, trace: Sequence[Request]) -> List[RequestRecord]:
        """Replays `trace`: hits in host segments, misses through the device greedy."""
        touch_c: List[int] = []
        touch_s: List[int] = []
        out = []
        for r in trace:
            if self.last_t is not None and r.t < self.last_t:
                raise A.AbiError(A.KVT_ETRACE, f"trace timestamps are not monotone (t={r.t} after t={self.last_t})")
            if r.n_new_tokens < 0:
                raise A.AbiError(A.KVT_ETRACE, f"negative n_new_tokens for context {r.context}")
            self.last_t = r.t
            c = self.arrays.index.get(r.context)
            if c is None:
                raise A.AbiError(A.KVT_ETRACE, f"trace names unknown context {r.context}")
            prof = self.prof[r.context]
            stamp = self.stamp
            self.stamp += 1
            ti = int(self.tier_index[c])
            if ti >= 0:  # hit (simulate.cpp:165-194)
                tier = self.tiers[ti]
                m, ratio = int(self.method[c]), float(self.ratio[c])
                name = self.names[m]
                load = load_time(compressed_size(prof.original_size_bytes, ratio), tier, self.ovh[m])
                ttft = load + prefill_time(r.n_new_tokens, self.sc.params) + 0.0
                truth = self.sc.truth.get(r.context)
                if truth is not None:
                    s_k = truth[name]
                    quality = synth_quality(s_k[0], s_k[1], ratio)
                else:
                    quality = quality_of(prof, name, ratio)
                rec = RequestRecord(r, True, tier.tier_id, name, ratio, ttft, quality)
                touch_c.append(c)
                touch_s.append(stamp)
            else:  # miss (simulate.cpp:195-222): recompute, then the joint store
                tokens = token_count(prof.original_size_bytes, self.sc.params) + r.n_new_tokens
                rec = RequestRecord(r, False, -1, "", 1.0, prefill_time(tokens, self.sc.params) + 0.0, 1.0)
                self._flush_touches(touch_c, touch_s)
                self._insert([c], [1], [stamp])
                self._refresh()
            out.append(rec)
        self._flush_touches(touch_c, touch_s)
        self.records.extend(out)
        return out

    def step(self, request: Request) -> RequestRecord:
        return self.run([request])[0]

    def _flush_touches(self, cs: List[int], ss: List[int]):
        if cs:
            c = np.asarray(cs, np.int32)
            s = np.asarray(ss, np.int64)
            self.eng.abi.check(self.eng.abi.store_touch_many(self.store.s, A.ptr(c), A.ptr(s), len(cs)))
            self.n_device_calls += 1
            cs.clear()
            ss.clear()

    def finish(self) -> ReplayResult:  # simulate.cpp:229-244
        placements: Dict[str, int] = {}
        for ti, tier in enumerate(self.tiers):
            idx = np.nonzero(self.tier_index == ti)[0]
            for c in idx[np.argsort(self.seq[idx], kind="stable")]:
                key = "tier%d:%s@%s" % (tier.tier_id, self.names[int(self.method[c])],
                                        "%.6g" % float(self.ratio[c]))
                placements[key] = placements.get(key, 0) + 1
        return ReplayResult(list(self.records), aggregate(self.records), placements, list(self.actions))


def _nearest_rank(sorted_v: List[float], pct: float) -> float:  # simulate.cpp:255-261
    if not sorted_v:
        return 0.0
    rank = math.ceil(pct / 100.0 * float(len(sorted_v)))
    return sorted_v[min(int(max(rank, 1.0)) - 1, len(sorted_v) - 1)]


def aggregate(records: Sequence[RequestRecord]) -> Dict[str, object]:  # simulate.cpp:266-298
    m: Dict[str, object] = {"n_requests": len(records), "sum_ttft": 0.0, "mean_ttft": 0.0, "p50_ttft": 0.0,
                            "p90_ttft": 0.0, "p99_ttft": 0.0, "mean_quality": 0.0, "miss_fraction": 0.0,
                            "hit_fraction_by_tier": {}}
    if not records:
        return m
    ttfts, qsum, misses, by_tier, s = [], 0.0, 0, {}, 0.0
    for r in records:
        s += r.ttft
        ttfts.append(r.ttft)
        qsum += r.quality
        if r.hit:
            by_tier[r.tier] = by_tier.get(r.tier, 0) + 1
        else:
            misses += 1
    ttfts.sort()
    n = float(len(records))
    m.update(sum_ttft=s, mean_ttft=s / n, p50_ttft=_nearest_rank(ttfts, 50.0), p90_ttft=_nearest_rank(ttfts, 90.0),
             p99_ttft=_nearest_rank(ttfts, 99.0), mean_quality=qsum / n, miss_fraction=misses / n,
             hit_fraction_by_tier={str(t): cnt / n for t, cnt in sorted(by_tier.items())})
    return m


def replay(eng: Engine, scenario: Scenario, trace: Sequence[Request]) -> ReplayResult:
    """kvtier::replay (simulate.cpp:246-251) on the device store."""
    rp = Replayer(eng, scenario)
    rp.run(trace)
    return rp.finish()


__all__ = ["Request", "RequestRecord", "ReplayResult", "Scenario", "Replayer", "replay", "aggregate"]
