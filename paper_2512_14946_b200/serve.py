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

With drift tracking on (`maybe_reprofile`,
simulate.cpp:102-128; quality.cpp:158-220) or `miss_store_bottom`, a
request can change the profiles and reshuffle the whole store, so the loop
runs request by request: a re-profile rebuilds the context's quality table
from its truth curve (std::mt19937_64 noise, bit-exact), uploads the new
profile set and runs `rearrange` on the device. The LRU / fixed / impress /
prefill baselines (`Policy::parse`) run the same request-by-request loop with
their LRU cascade (placement.cpp:374-438) on the device store.
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
    profiling_windows: List[Tuple[float, float, float]] = field(default_factory=list)  # (start, duration, penalty)
    reprofile_count: int = 0


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
    seed: int = 0
    drift_config: Dict[str, float] = field(default_factory=dict)  # DriftConfig + ReprofileConfig
    policy: str = "joint"  # Policy::label(): joint, joint-qargmax, lru, fixed:<m>:<r>, impress:<f>[:<o>], prefill

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
                      doc.get("rule", "utility"), int(doc.get("seed", 0)), dict(doc.get("drift_config") or {}),
                      doc.get("policy", "joint"))
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


def parse_policy(text: str):  # placement.cpp:440-495 Policy::parse -> (kind, (method, ratio), chunk overhead)
    parts = text.split(":")
    head = parts[0]
    bad = A.ValidationError(A.KVT_EVALIDATION, f"unknown policy '{text}'")
    if head in ("joint", "joint-qargmax", "lru", "prefill"):
        if len(parts) != 1:
            raise bad
        return ("joint" if head.startswith("joint") else head), None, 1.3
    if head == "fixed" and len(parts) == 3:
        r = float(parts[2])
        if not parts[1] or not (0.0 < r <= 1.0):
            raise A.ValidationError(A.KVT_EVALIDATION, "fixed ratio must be in (0, 1]")
        return "fixed", (parts[1], r), 1.3
    if head == "impress" and len(parts) in (2, 3):
        f = float(parts[1])
        o = float(parts[2]) if len(parts) == 3 else 1.3
        if not (0.0 < f <= 1.0) or not o > 0.0:
            raise A.ValidationError(A.KVT_EVALIDATION, "impress keep fraction must be in (0, 1]")
        return "impress", (None, f), o
    raise bad


class MT19937_64:
    """std::mt19937_64 (C++11 [rand.predef]; the reference's Rng engine,
    proj/include/kvtier/rng.hpp), bit-exact."""
    _MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        mt = [seed & self._MASK]
        for i in range(1, 312):
            mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & self._MASK)
        self.mt, self.i = mt, 312

    def next_u64(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                x = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                xa = (x >> 1) ^ (0xB5026F5AA96619E9 if x & 1 else 0)
                mt[k] = mt[(k + 156) % 312] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self._MASK

    def uniform(self, lo: float, hi: float) -> float:  # rng.hpp uniform01 / uniform
        return lo + (hi - lo) * (float(self.next_u64() >> 11) * 2.0 ** -53)


@dataclass
class DriftState:  # proj/include/kvtier/quality.hpp:62-72
    window_size: int = 0
    observed_sum: float = 0.0
    profiled_sum: float = 0.0
    n_observations: int = 0
    window: List[Tuple[float, float]] = field(default_factory=list)

    def _n(self) -> int:
        return self.n_observations if self.window_size == 0 else len(self.window)

    def observed_mean(self) -> float:
        n = self._n()
        return 0.0 if n == 0 else self.observed_sum / float(n)

    def profiled_mean(self) -> float:
        n = self._n()
        return 0.0 if n == 0 else self.profiled_sum / float(n)

    def record(self, predicted: float, observed: float):  # quality.cpp:158-180 record_observation
        if self.window_size == 0:
            self.profiled_sum += predicted
            self.observed_sum += observed
            self.n_observations += 1
            return
        self.window.append((predicted, observed))
        if len(self.window) > self.window_size:
            self.window.pop(0)
        self.profiled_sum = 0.0
        self.observed_sum = 0.0
        for pr, ob in self.window:
            self.profiled_sum += pr
            self.observed_sum += ob
        self.n_observations += 1


def reprofile(old: ContextProfile, truth: Dict[str, Tuple[float, float]], noise_seed: int,
              noise: float) -> ContextProfile:  # proj/src/quality.cpp:191-220
    rng = MT19937_64(noise_seed)
    table = {}
    for m in sorted(old.quality_table, key=lambda x: x.encode()):  # std::map order
        values = list(old.quality_table[m])
        curve = truth.get(m)
        for i, r in enumerate(old.ratio_grid):
            q = synth_quality(curve[0], curve[1], r) if curve is not None else values[i]
            if noise > 0.0:
                q += rng.uniform(-noise, noise)
            values[i] = min(max(q, 0.0), 1.0)
        for i in range(1, len(values)):
            values[i] = max(values[i], values[i - 1])
        values[-1] = 1.0
        table[m] = values
    return ContextProfile(old.context, old.original_size_bytes, old.frequency, list(old.ratio_grid), table)


class Replayer:
    """kvtier::Replayer (joint policy) on the device store."""

    def __init__(self, eng: Engine, scenario: Scenario):
        self.sc = scenario
        self.eng = eng
        self.tiers = sorted_tiers(scenario.tiers)  # Replayer keeps the validated order
        self.arrays = ProfileArrays.from_profiles(scenario.profiles, scenario.space)
        self.prof = {p.context: p for p in scenario.profiles}
        self.ps = eng.pset(self.arrays)
        self.store = eng.store(self.tiers, self.arrays.n, scenario.space)
        self.rule = A.KVT_RULE_UTILITY if scenario.rule == "utility" else A.KVT_RULE_QUALITY_FIRST
        self.kind, self.fixed, self.chunk_overhead = parse_policy(scenario.policy)
        if self.kind == "joint" and scenario.policy == "joint-qargmax":
            self.rule = A.KVT_RULE_QUALITY_FIRST
        self.names = scenario.space.method_names
        self.ovh = [m.decompression_overhead for m in scenario.space.methods]
        self.stamp = 0
        self.actions: List[Tuple[str, str, int, str, float]] = []
        self.records: List[RequestRecord] = []
        self.last_t: Optional[float] = None
        self.n_device_calls = 0
        self._qcache: Dict[Tuple[int, int, float], float] = {}
        dc = scenario.drift_config
        self.window_size = int(dc.get("window_size", 0))
        self.drift_states: Dict[int, DriftState] = {}
        self.windows: List[Tuple[float, float, float]] = []  # (start, duration, penalty)
        self.reprofile_count = 0
        self.arrivals: List[float] = []
        self._arr_lo = 0
        self.rp_rng = MT19937_64((scenario.seed ^ 0x9E3779B97F4A7C15) & MT19937_64._MASK)
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

    def _insert_ops(self, ctx: Sequence[int], stamps: Sequence[int]) -> List[np.ndarray]:
        """insert_joint of every miss (frequency 1) in one call; the action
        list split per op (each op starts with its Insert action)."""
        if not ctx:
            return []
        n0 = len(self.actions)
        acts = self.store.insert_joint(self.ps, self.sc.space, self.sc.params, np.asarray(ctx, np.int32),
                                       frequency=np.ones(len(ctx), np.int64), stamp=np.asarray(stamps, np.int64),
                                       rule=self.rule)
        self.n_device_calls += 1
        ids = self.arrays.ids
        for a in acts:
            self.actions.append((KIND_NAMES[int(a["kind"])], ids[int(a["ctx"])], int(a["tier_id"]),
                                 self.names[int(a["method"])], float(a["ratio"])))
        starts = np.nonzero(acts["kind"] == A.KVT_INSERT)[0]
        assert len(starts) == len(ctx) and len(self.actions) - n0 == len(acts)
        return np.split(acts, starts[1:])

    def _apply(self, acts: np.ndarray):
        """Replays one op's actions (placement.cpp:213-221, 225-250) on the mirror."""
        tix = {t.tier_id: i for i, t in enumerate(self.tiers)}
        for a in acts:
            c = int(a["ctx"])
            ti = tix[int(a["tier_id"])]
            if int(a["kind"]) != A.KVT_RECOMPRESS and int(self.tier_index[c]) != ti:
                self._seq += 1
                self.seq[c] = self._seq  # arrival order within the tier
            self.tier_index[c] = ti
            self.method[c] = int(a["method"])
            self.ratio[c] = float(a["ratio"])

    def _refresh(self):
        snap = self.store.snapshot()
        self.tier_index = snap["tier_index"].astype(np.int64)
        self.method = snap["method"].astype(np.int64)
        self.ratio = snap["ratio"].astype(np.float64)
        self.seq = snap["seq"].astype(np.int64)
        self._seq = int(self.seq.max()) if len(self.seq) else 0

    def _warm_up(self):  # simulate.cpp:72-85: every context, frequency 0, one stamp each
        order = self.sc.order or sorted(self.prof, key=lambda c: c.encode())
        ctx = [self.arrays.index[c] for c in order]
        stamps = list(range(self.stamp, self.stamp + len(ctx)))
        self.stamp += len(ctx)
        if self.kind == "joint":
            self._insert(ctx, [0] * len(ctx), stamps)
        else:
            for c, st in zip(ctx, stamps):
                self._policy_insert(c, 0, st)

    # -- the baselines (placement.cpp:374-438, 515-547): a store at the top
    # tier at one fixed configuration, overflow pushes the least recently
    # used entry one tier down, unchanged (on the device store)
    def _policy_insert(self, c: int, freq: int, stamp: int):
        if self.kind == "joint":
            self._insert([c], [freq], [stamp])
            return
        if self.kind == "prefill":
            return
        if self.kind == "lru":
            m, ratio = 0, 1.0
        elif self.kind == "fixed":
            if self.fixed[0] not in self.names:
                raise A.ValidationError(A.KVT_EVALIDATION, f"fixed policy method {self.fixed[0]} is not in the method set")
            m, ratio = self.names.index(self.fixed[0]), self.fixed[1]
        else:  # impress: (first method, keep fraction)
            m, ratio = 0, self.fixed[1]
        cid = self.arrays.ids[c]
        orig = self.prof[cid].original_size_bytes
        self.store.add(c, 0, m, ratio, orig, freq, stamp)
        self.actions.append(("insert", cid, self.tiers[0].tier_id, self.names[m], ratio))
        self.n_device_calls += 1
        for ti in range(len(self.tiers)):
            while True:
                occ = self.store.occupancy()
                cap = self.tiers[ti].capacity_bytes
                if cap is None or occ[ti] <= cap:
                    break
                if ti + 1 >= len(self.tiers):
                    raise A.ValidationError(A.KVT_EVALIDATION,
                                            f"tier {self.tiers[ti].name} overflows and there is no lower tier")
                snap = self.store.snapshot()
                idx = np.nonzero(snap["tier_index"] == ti)[0]
                idx = idx[np.argsort(snap["seq"][idx], kind="stable")]  # arrival order
                v = int(idx[np.argmin(snap["last_access"][idx])])  # first minimum, like the reference
                e = self.store.remove(v)
                self.store.add(v, ti + 1, int(e.method), float(e.ratio), int(e.original_size_bytes),
                               int(e.frequency), int(e.last_access))
                self.actions.append(("evict", self.arrays.ids[v], self.tiers[ti + 1].tier_id, self.names[int(e.method)],
                                     float(e.ratio)))
                self.n_device_calls += 4

    # -- serving
    def _quality(self, c: int, m: int, ratio: float) -> float:
        """Achieved quality of context c served at (m, ratio): the truth curve
        when the scenario has one, else the profile (simulate.cpp:179-184)."""
        key = (c, m, ratio)
        q = self._qcache.get(key)
        if q is None:
            cid = self.arrays.ids[c]
            truth = self.sc.truth.get(cid)
            name = self.names[m]
            q = synth_quality(*truth[name], ratio) if truth is not None else quality_of(self.prof[cid], name, ratio)
            self._qcache[key] = q
        return q

    def run(self, trace: Sequence[Request]) -> List[RequestRecord]:
        """Replays `trace`. A joint-policy store never drops a context (the
        bottom tier is unlimited), so the misses are the first requests of
        the contexts not yet resident; the hits between two misses are served
        as one vectorised segment from the placement mirror, with one batched
        touch, and each miss runs insert_joint on the device store."""
        n = len(trace)
        if n == 0:
            return []
        if self.sc.drift or self.sc.miss_store_bottom or self.kind != "joint":
            return self._run_sequential(trace)
        t = np.fromiter((r.t for r in trace), np.float64, n)
        nnew = np.fromiter((r.n_new_tokens for r in trace), np.int64, n)
        try:
            ctx = np.fromiter((self.arrays.index[r.context] for r in trace), np.int64, n)
        except KeyError as e:
            raise A.AbiError(A.KVT_ETRACE, f"trace names unknown context {e.args[0]}") from None
        prev = np.concatenate([[self.last_t if self.last_t is not None else -np.inf], t[:-1]])
        bad = np.nonzero(t < prev)[0]
        if len(bad):
            k = int(bad[0])
            raise A.AbiError(A.KVT_ETRACE, f"trace timestamps are not monotone (t={t[k]} after t={prev[k]})")
        neg = np.nonzero(nnew < 0)[0]
        if len(neg):
            raise A.AbiError(A.KVT_ETRACE, f"negative n_new_tokens for context {trace[int(neg[0])].context}")
        self.last_t = float(t[-1])
        stamps = self.stamp + np.arange(n, dtype=np.int64)
        self.stamp += n
        # misses: first request of every context that is not resident yet
        resident = self.tier_index[ctx] >= 0
        _, first = np.unique(ctx, return_index=True)
        is_first = np.zeros(n, bool)
        is_first[first] = True
        miss_at = np.nonzero(is_first & ~resident)[0]

        hit = np.ones(n, bool)
        tier_id = np.full(n, -1, np.int64)
        meth = np.full(n, -1, np.int64)
        ratio = np.ones(n, np.float64)
        ttft = np.zeros(n, np.float64)
        qual = np.ones(n, np.float64)
        p = self.sc.params
        tier_lat = np.array([x.fixed_access_latency for x in self.tiers], np.float64)
        tier_bw = np.array([x.read_bandwidth for x in self.tiers], np.float64)
        tier_ids = np.array([x.tier_id for x in self.tiers], np.int64)
        ovh = np.asarray(self.ovh, np.float64)
        orig = self.arrays.orig

        def serve_hits(lo, hi):
            if hi <= lo:
                return
            c = ctx[lo:hi]
            ti = self.tier_index[c]
            m = self.method[c]
            r = self.ratio[c]
            # simulate.cpp:165-178: load + prefill(new tokens) + penalty (no re-profiling windows)
            size = np.maximum(1.0, np.floor(orig[c].astype(np.float64) * r + 0.5))
            load = tier_lat[ti] + size / tier_bw[ti] + size * ovh[m]
            nn = nnew[lo:hi].astype(np.float64)
            ttft[lo:hi] = (load + (p.prefill_a * nn + p.prefill_b * nn * nn)) + 0.0
            tier_id[lo:hi] = tier_ids[ti]
            meth[lo:hi] = m
            ratio[lo:hi] = r
            qual[lo:hi] = [self._quality(int(a), int(b), float(x)) for a, b, x in zip(c, m, r)]

        # every miss's store in ONE device call: insert_joint runs the ops in
        # order (each op = an insert + its overflow cascade, the same state
        # evolution as one call per miss); touches never steer the joint
        # policy (utility uses the profile frequency), so the hits between
        # two misses are served from the mirror as it stood after the
        # earlier op, replayed on the host from the action list
        ops = self._insert_ops([int(ctx[j]) for j in miss_at], [int(stamps[j]) for j in miss_at])
        lo = 0
        for k, j in enumerate(miss_at):
            j = int(j)
            serve_hits(lo, j)
            c = int(ctx[j])
            # simulate.cpp:195-203: recompute the whole context, lossless; then the joint store
            tokens = token_count(int(orig[c]), p) + int(nnew[j])
            nt = float(tokens)
            hit[j] = False
            ttft[j] = (p.prefill_a * nt + p.prefill_b * nt * nt) + 0.0
            self._apply(ops[k])
            lo = j + 1
        serve_hits(lo, n)
        if len(miss_at):
            self._refresh()  # the device store is the source of truth again
        # the hits' touches, in order, after the inserts they follow (a context is
        # only ever touched after its own insert, so freq / last_access end equal)
        if hit.any():
            cc = np.ascontiguousarray(ctx[hit], np.int32)
            ss = np.ascontiguousarray(stamps[hit])
            self.eng.abi.check(self.eng.abi.store_touch_many(self.store.s, A.ptr(cc), A.ptr(ss), len(cc)))
            self.n_device_calls += 1
        out = [RequestRecord(trace[i], bool(hit[i]), int(tier_id[i]), self.names[int(meth[i])] if hit[i] else "",
                             float(ratio[i]), float(ttft[i]), float(qual[i])) for i in range(n)]
        self.records.extend(out)
        return out

    # -- request by request (drift tracking / re-profiling, miss_store_bottom)
    def _gpu_free(self, now: float) -> bool:  # simulate.cpp:88-93
        gw = float(self.sc.drift_config.get("gpu_window", 1.0))
        while self._arr_lo < len(self.arrivals) and self.arrivals[self._arr_lo] <= now - gw:
            self._arr_lo += 1
        return len(self.arrivals) - self._arr_lo < int(self.sc.drift_config.get("max_batch", 8))

    def _active_penalty(self, now: float) -> float:  # simulate.cpp:95-100
        pen = 0.0
        for start, dur, p in self.windows:
            if now >= start and now < start + dur:
                pen += p
        return pen

    def _upload_profiles(self):
        self.arrays = ProfileArrays.from_profiles(list(self.prof.values()), self.sc.space)
        self.ps = self.eng.pset(self.arrays)
        self._qcache.clear()

    def _maybe_reprofile(self, c: int, now: float):  # simulate.cpp:102-128
        if not self.sc.drift or self.kind != "joint":
            return
        st = self.drift_states.get(c)
        if st is None:
            return
        dc = self.sc.drift_config
        thr = float(dc.get("threshold", 0.3))
        if not (self._gpu_free(now) and st.n_observations >= int(dc.get("min_samples", 10))
                and (st.profiled_mean() - st.observed_mean()) > thr):  # quality.cpp:182-189 should_reprofile
            return
        cid = self.arrays.ids[c]
        truth = self.sc.truth.get(cid)
        if truth is None:
            return
        seed = self.rp_rng.next_u64()
        self.prof[cid] = reprofile(self.prof[cid], truth, seed, float(dc.get("noise_amplitude", 0.0)))
        self.windows.append((now, float(dc.get("duration", 2.0)), float(dc.get("penalty", 0.5))))
        self.reprofile_count += 1
        self.drift_states[c] = DriftState(self.window_size)
        self._upload_profiles()
        self._record_actions(self.store.rearrange(self.ps, self.sc.space, self.sc.params, rule=self.rule))
        self.n_device_calls += 1
        self._refresh()

    def _record_actions(self, acts):
        ids = self.arrays.ids
        for a in acts:
            self.actions.append((KIND_NAMES[int(a["kind"])], ids[int(a["ctx"])], int(a["tier_id"]),
                                 self.names[int(a["method"])], float(a["ratio"])))

    def _run_sequential(self, trace: Sequence[Request]) -> List[RequestRecord]:
        p = self.sc.params
        out: List[RequestRecord] = []
        touch_c: List[int] = []
        touch_s: List[int] = []
        for r in trace:
            if self.last_t is not None and r.t < self.last_t:
                raise A.AbiError(A.KVT_ETRACE, f"trace timestamps are not monotone (t={r.t} after t={self.last_t})")
            if r.n_new_tokens < 0:
                raise A.AbiError(A.KVT_ETRACE, f"negative n_new_tokens for context {r.context}")
            self.last_t = r.t
            self.arrivals.append(r.t)
            c = self.arrays.index.get(r.context)
            if c is None:
                raise A.AbiError(A.KVT_ETRACE, f"trace names unknown context {r.context}")
            prof = self.prof[r.context]
            stamp = self.stamp
            self.stamp += 1
            penalty = self._active_penalty(r.t)
            ti = int(self.tier_index[c])
            if ti >= 0:  # hit
                tier = self.tiers[ti]
                m, ratio = int(self.method[c]), float(self.ratio[c])
                name = self.names[m]
                load = load_time(compressed_size(prof.original_size_bytes, ratio), tier, self.ovh[m])
                if self.kind == "impress":
                    load *= self.chunk_overhead  # chunked reads amplify the fetch (simulate.cpp:170-172)
                ttft = load + prefill_time(r.n_new_tokens, p) + penalty
                predicted = quality_of(prof, name, ratio)
                truth = self.sc.truth.get(r.context)
                achieved = synth_quality(*truth[name], ratio) if truth is not None else predicted
                rec = RequestRecord(r, True, tier.tier_id, name, ratio, ttft, achieved)
                touch_c.append(c)
                touch_s.append(stamp)
                if self.sc.drift and self.kind == "joint" and truth is not None:  # simulate.cpp:186-193
                    self.drift_states.setdefault(c, DriftState(self.window_size)).record(predicted, achieved)
            else:  # miss
                tokens = token_count(prof.original_size_bytes, p) + r.n_new_tokens
                rec = RequestRecord(r, False, -1, "", 1.0, prefill_time(tokens, p) + penalty, 1.0)
                self._touch(touch_c, touch_s)  # LRU reads last_access
                if self.sc.miss_store_bottom and self.kind == "joint":  # simulate.cpp:203-216: bottom tier, rearrange
                    bottom = len(self.tiers) - 1
                    self.store.add(c, bottom, 0, 1.0, prof.original_size_bytes, 1, stamp)
                    self.actions.append(("insert", r.context, self.tiers[bottom].tier_id, self.names[0], 1.0))
                    self._record_actions(self.store.rearrange(self.ps, self.sc.space, self.sc.params, rule=self.rule))
                    self.n_device_calls += 2
                elif self.kind == "joint":
                    self._insert([c], [1], [stamp])
                else:
                    self._policy_insert(c, 1, stamp)
                self._refresh()
            out.append(rec)
            if self.sc.drift:
                self._touch(touch_c, touch_s)  # a re-profile's rearrange re-inserts with the touched stats
                self._maybe_reprofile(c, r.t)
        self._touch(touch_c, touch_s)
        self.records.extend(out)
        return out

    def _touch(self, cs: List[int], ss: List[int]):
        if cs:
            cc = np.asarray(cs, np.int32)
            st = np.asarray(ss, np.int64)
            self.eng.abi.check(self.eng.abi.store_touch_many(self.store.s, A.ptr(cc), A.ptr(st), len(cs)))
            self.n_device_calls += 1
            cs.clear()
            ss.clear()

    def step(self, request: Request) -> RequestRecord:
        return self.run([request])[0]

    def finish(self) -> ReplayResult:  # simulate.cpp:229-244
        placements: Dict[str, int] = {}
        for ti, tier in enumerate(self.tiers):
            idx = np.nonzero(self.tier_index == ti)[0]
            for c in idx[np.argsort(self.seq[idx], kind="stable")]:
                key = "tier%d:%s@%s" % (tier.tier_id, self.names[int(self.method[c])],
                                        "%.6g" % float(self.ratio[c]))
                placements[key] = placements.get(key, 0) + 1
        return ReplayResult(list(self.records), aggregate(self.records), placements, list(self.actions),
                            list(self.windows), self.reprofile_count)


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
