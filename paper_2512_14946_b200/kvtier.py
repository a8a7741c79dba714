"""Python mirror of the reference's placement interface (namespace kvtier,
proj/include/kvtier/{core,quality,utility,placement}.hpp) over the C ABI.

The names follow the reference so the parity tests read like its doctest
suites: TierSpec, CompressionMethod, CandidateSpace, ContextProfile,
UtilityParams, score_candidates (= all_candidates for every context),
best_config, StoreState.insert_joint / resolve_overflow / rearrange /
least_drop_update / placement_utility. Errors raise ValidationError exactly
where the reference throws kvtier::ValidationError.

`Engine(abi)` works with any implementation of the ABI; the product engine
is `Engine(paper_2512_14946_b200.product())` (CUDA, fails loudly without the
built extension).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence

import numpy as np

from . import _abi as A
from ._abi import ValidationError  # noqa: F401  (re-export)


@dataclass
class TierSpec:  # proj/include/kvtier/core.hpp:63-71
    tier_id: int
    name: str = ""
    capacity_bytes: Optional[int] = None  # None = unlimited
    read_bandwidth: float = 1.0
    fixed_access_latency: float = 0.0


@dataclass
class CompressionMethod:  # proj/include/kvtier/core.hpp:28-31
    name: str
    decompression_overhead: float = 0.0


DEFAULT_METHODS = ("keydiff", "knorm", "snapkv")  # proj/src/core.cpp:29-31
DEFAULT_RATIO_GRID = (0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 1.0)  # proj/src/utility.cpp:39-41


class CandidateSpace:  # proj/include/kvtier/utility.hpp:31-46
    def __init__(self, methods: Sequence, ratio_grid: Sequence[float]):
        self.methods = [m if isinstance(m, CompressionMethod) else CompressionMethod(m) for m in methods]
        self.raw_ratios = [float(r) for r in ratio_grid]
        # enumeration order: unique, descending (proj/src/utility.cpp:31-32)
        self.ratios = sorted(set(self.raw_ratios), reverse=True)
        self._names = (C.c_char_p * len(self.methods))(*[m.name.encode() for m in self.methods])
        self._ovh = (C.c_double * len(self.methods))(*[m.decompression_overhead for m in self.methods])
        self._ratios = (C.c_double * len(self.raw_ratios))(*self.raw_ratios)
        self.c = A.Space(len(self.methods), self._names, self._ovh, len(self.raw_ratios), self._ratios)

    @staticmethod
    def default_space() -> "CandidateSpace":
        return CandidateSpace(DEFAULT_METHODS, DEFAULT_RATIO_GRID)

    @property
    def method_names(self) -> List[str]:
        return [m.name for m in self.methods]

    def method_index(self, name: str) -> int:
        return self.method_names.index(name)


@dataclass
class UtilityParams:  # proj/include/kvtier/core.hpp:74-79
    alpha: float = 1.0
    prefill_a: float = 2e-5
    prefill_b: float = 1e-10
    bytes_per_token: float = 1.2e5

    @property
    def c(self):
        return A.Params(self.alpha)


@dataclass
class ContextProfile:  # proj/include/kvtier/quality.hpp:20-29
    context: str
    original_size_bytes: int
    frequency: float = 1.0
    ratio_grid: List[float] = field(default_factory=list)
    quality_table: Dict[str, List[float]] = field(default_factory=dict)


def _tiers_c(tiers: Sequence[TierSpec]):
    arr = (A.Tier * len(tiers))()
    for i, t in enumerate(tiers):
        arr[i] = A.Tier(int(t.tier_id), 1 if t.capacity_bytes is None else 0,
                        0 if t.capacity_bytes is None else int(t.capacity_bytes),
                        float(t.read_bandwidth), float(t.fixed_access_latency))
    return arr


def sorted_tiers(tiers: Sequence[TierSpec]) -> List[TierSpec]:
    return sorted(tiers, key=lambda t: t.tier_id)  # stable, like validate_hierarchy


class ProfileArrays:
    """Struct-of-arrays form of a ProfileMap (kvt_profiles) for one space.

    Contexts are ordered by byte-lexicographic id (std::map order)."""

    def __init__(self, ids, orig, freq, goff, grid, qual, has):
        self.ids = list(ids)
        self.orig = np.ascontiguousarray(orig, dtype=np.int64)
        self.freq = np.ascontiguousarray(freq, dtype=np.float64)
        self.goff = np.ascontiguousarray(goff, dtype=np.int32)
        self.grid = np.ascontiguousarray(grid, dtype=np.float64)
        self.qual = np.ascontiguousarray(qual, dtype=np.float64)
        self.has = np.ascontiguousarray(has, dtype=np.uint8)
        self.n = len(self.orig)
        self.M = self.has.shape[1] if self.has.ndim == 2 else 0
        self.index = {cid: i for i, cid in enumerate(self.ids)}

    @staticmethod
    def from_profiles(profiles: Iterable[ContextProfile], space: CandidateSpace) -> "ProfileArrays":
        profs = sorted(profiles, key=lambda p: p.context.encode())
        names = space.method_names
        M = len(names)
        orig, freq, goff, grid, qual = [], [], [0], [], []
        has = np.zeros((len(profs), M), np.uint8)
        for c, p in enumerate(profs):
            g = [float(x) for x in p.ratio_grid]
            orig.append(int(p.original_size_bytes))
            freq.append(float(p.frequency))
            grid.extend(g)
            goff.append(len(grid))
            for m, nm in enumerate(names):
                row = p.quality_table.get(nm)
                if row is None:
                    qual.extend([0.0] * len(g))
                else:
                    has[c, m] = 1
                    qual.extend(float(x) for x in row)
        return ProfileArrays([p.context for p in profs], orig, freq, goff, grid, qual, has)

    @staticmethod
    def uniform_grid(ids, orig, freq, grid, qual_nmg, has=None) -> "ProfileArrays":
        """Fast path: every context shares one grid; qual_nmg is [n][M][G]."""
        n, M, G = qual_nmg.shape
        goff = np.arange(n + 1, dtype=np.int32) * G
        if has is None:
            has = np.ones((n, M), np.uint8)
        return ProfileArrays(ids, orig, freq, goff, np.tile(np.asarray(grid, np.float64), n),
                             np.ascontiguousarray(qual_nmg, np.float64).reshape(-1), has)

    def c_struct(self):
        return A.Profiles(
            self.n, self.M,
            self.orig.ctypes.data_as(C.POINTER(C.c_int64)),
            self.freq.ctypes.data_as(C.POINTER(C.c_double)),
            self.goff.ctypes.data_as(C.POINTER(C.c_int32)),
            self.grid.ctypes.data_as(C.POINTER(C.c_double)),
            self.qual.ctypes.data_as(C.POINTER(C.c_double)),
            self.has.ctypes.data_as(C.POINTER(C.c_uint8)))


class Engine:
    """One ABI implementation + a handle (device stream for the CUDA one)."""

    def __init__(self, abi: A.Abi, device: int = 0, stream: int = 0):
        self.abi = abi
        h = C.c_void_p()
        abi.check(abi.create(device, stream or None, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.abi.destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- profiles
    def pset(self, arrays: ProfileArrays) -> "PSet":
        return PSet(self, arrays)

    # -- utility.cpp:129-145 all_candidates, dense over contexts
    def score_candidates(self, ps: "PSet", tiers, space: CandidateSpace, params: UtilityParams):
        n, T, M, R = ps.arrays.n, len(tiers), len(space.methods), len(space.ratios)
        size = np.zeros((n, R), np.int64)
        qual = np.zeros((n, M, R), np.float64)
        valid = np.zeros((n, M, R), np.uint8)
        ttft = np.zeros((n, T, M, R), np.float64)
        util = np.zeros((n, T, M, R), np.float64)
        tc = _tiers_c(tiers)
        self.abi.check(self.abi.score_candidates(self.h, ps.p, tc, T, C.byref(space.c), C.byref(params.c),
                                                 A.ptr(size), A.ptr(qual), A.ptr(valid), A.ptr(ttft),
                                                 A.ptr(util)))
        return dict(size=size, quality=qual, valid=valid, ttft=ttft, utility=util)

    # -- utility.cpp:159-172 best_config for every context
    def best_config(self, ps: "PSet", tiers, space: CandidateSpace, params: UtilityParams,
                    rule: int = A.KVT_RULE_UTILITY):
        out = np.zeros(ps.arrays.n, A.BEST_DTYPE)
        tc = _tiers_c(tiers)
        self.abi.check(self.abi.best_config(self.h, ps.p, tc, len(tiers), C.byref(space.c),
                                            C.byref(params.c), rule, A.ptr(out)))
        return out

    def oracle_mckp(self, ps: "PSet", tiers, space: CandidateSpace, params: UtilityParams,
                    max_assignments: float = 1e7):
        """oracle_mckp (proj/src/placement.cpp:300-372): the exact
        one-configuration-per-context optimum; (total utility, BEST_DTYPE[n])."""
        out = np.zeros(ps.arrays.n, A.BEST_DTYPE)
        total = C.c_double()
        tc = _tiers_c(tiers)
        self.abi.check(self.abi.oracle_mckp(self.h, ps.p, tc, len(tiers), C.byref(space.c), C.byref(params.c),
                                            float(max_assignments), C.byref(total), A.ptr(out)))
        return total.value, out

    def store(self, tiers, n_ctx: int, space: Optional[CandidateSpace] = None) -> "StoreState":
        return StoreState(self, tiers, n_ctx, space)


class PSet:
    def __init__(self, eng: Engine, arrays: ProfileArrays):
        self.eng = eng
        self.arrays = arrays
        p = C.c_void_p()
        st = arrays.c_struct()
        eng.abi.check(eng.abi.pset_create(eng.h, C.byref(st), C.byref(p)))
        self.p = p

    def __del__(self):
        try:
            if self.p:
                self.eng.abi.pset_destroy(self.p)
        except Exception:
            pass


class MergedPSet(PSet):
    """A profile set assembled on the device from gathered rank records
    (kvt_pset_merge); refilled in place by later merges of the same size."""

    class _Dims:
        def __init__(self, n):
            self.n = n

    def __init__(self, eng: Engine, n_total: int):  # noqa: super().__init__ uploads host rows; not here
        self.eng = eng
        self.arrays = MergedPSet._Dims(n_total)
        self.p = C.c_void_p()

    def merge(self, records, world: int, n_ctx: int, grid_len: int, n_methods: int) -> "MergedPSet":
        self.eng.abi.check(self.eng.abi.pset_merge(self.eng.h, A.ptr(records), world, n_ctx, grid_len, n_methods,
                                                   C.byref(self.p)))
        return self


class StoreState:  # proj/include/kvtier/placement.hpp:29-70
    def __init__(self, eng: Engine, tiers: Sequence[TierSpec], n_ctx: int,
                 space: Optional[CandidateSpace] = None):
        self.eng = eng
        self.abi = eng.abi
        self.tiers = sorted_tiers(tiers)
        self.n_ctx = n_ctx
        s = C.c_void_p()
        tc = _tiers_c(tiers)
        self.abi.check(self.abi.store_create(eng.h, tc, len(tiers), n_ctx, C.byref(s)))
        self.s = s
        if space is not None:
            self.bind_space(space)

    def __del__(self):
        try:
            if self.s:
                self.abi.store_destroy(self.s)
        except Exception:
            pass

    def bind_space(self, space: CandidateSpace):
        self.abi.check(self.abi.store_bind_space(self.s, C.byref(space.c)))

    def _actions(self, n: int) -> np.ndarray:
        out = np.zeros(n, A.ACTION_DTYPE)
        if n:
            self.abi.check(self.abi.store_actions(self.s, A.ptr(out), n))
        return out

    def add(self, ctx: int, tier_index: int, method: int, ratio: float, original_size_bytes: int,
            frequency: int = 0, last_access: int = 0):
        e = A.Entry(tier_index, method, ratio, original_size_bytes, frequency, last_access, 0)
        self.abi.check(self.abi.store_add(self.s, ctx, C.byref(e)))

    def remove(self, ctx: int):
        e = A.Entry()
        self.abi.check(self.abi.store_remove(self.s, ctx, C.byref(e)))
        return e

    def reconfigure(self, ctx: int, method: int, ratio: float):
        self.abi.check(self.abi.store_reconfigure(self.s, ctx, method, ratio))

    def touch(self, ctx: int, stamp: int):
        self.abi.check(self.abi.store_touch(self.s, ctx, stamp))

    def clear(self):
        self.abi.check(self.abi.store_clear(self.s))

    def occupancy(self) -> np.ndarray:
        occ = np.zeros(len(self.tiers), np.int64)
        self.abi.check(self.abi.store_occupancy(self.s, A.ptr(occ)))
        return occ

    def snapshot(self) -> np.ndarray:
        out = np.zeros(self.n_ctx, A.ENTRY_DTYPE)
        self.abi.check(self.abi.store_snapshot(self.s, A.ptr(out)))
        return out

    def residents(self) -> List[List[int]]:
        """Per tier, context indices in arrival order (StoreState::residents)."""
        snap = self.snapshot()
        out = []
        for t in range(len(self.tiers)):
            idx = np.nonzero(snap["tier_index"] == t)[0]
            out.append(idx[np.argsort(snap["seq"][idx], kind="stable")].tolist())
        return out

    def first_over_capacity(self) -> Optional[int]:
        occ = self.occupancy()
        for i, t in enumerate(self.tiers):
            if t.capacity_bytes is not None and occ[i] > t.capacity_bytes:
                return i
        return None

    def least_drop_update(self, ps: PSet, space: CandidateSpace, params: UtilityParams,
                          tier_index: int) -> A.Update:
        u = A.Update()
        self.abi.check(self.abi.least_drop_update(self.s, ps.p, C.byref(space.c), C.byref(params.c),
                                                  tier_index, C.byref(u)))
        return u

    def resolve_overflow(self, ps: PSet, space: CandidateSpace, params: UtilityParams) -> np.ndarray:
        n = C.c_int64()
        rc = self.abi.resolve_overflow(self.s, ps.p, C.byref(space.c), C.byref(params.c), C.byref(n))
        acts = self._actions(n.value)
        self.abi.check(rc)
        return acts

    def insert_joint(self, ps: PSet, space: CandidateSpace, params: UtilityParams, ctx,
                     frequency=None, stamp=None, rule: int = A.KVT_RULE_UTILITY, cached: bool = False) -> np.ndarray:
        """insert_joint of every context of `ctx`, in order. cached=True runs
        the CPU cached-greedy baseline (ref_insert_joint_cached; reference
        library only)."""
        fn = self.abi.insert_joint_cached if cached else self.abi.insert_joint
        ctx = np.atleast_1d(np.asarray(ctx, np.int32))
        nops = len(ctx)
        freq = np.zeros(nops, np.int64) if frequency is None else np.atleast_1d(np.asarray(frequency, np.int64))
        stp = np.zeros(nops, np.int64) if stamp is None else np.atleast_1d(np.asarray(stamp, np.int64))
        n, done = C.c_int64(), C.c_int64()
        rc = fn(self.s, ps.p, C.byref(space.c), C.byref(params.c), rule,
                A.ptr(ctx), A.ptr(freq), A.ptr(stp), nops, C.byref(n), C.byref(done))
        self.last_done = done.value
        acts = self._actions(n.value)
        self.abi.check(rc)
        return acts

    def rearrange(self, ps: PSet, space: CandidateSpace, params: UtilityParams,
                  rule: int = A.KVT_RULE_UTILITY) -> np.ndarray:
        n = C.c_int64()
        rc = self.abi.rearrange(self.s, ps.p, C.byref(space.c), C.byref(params.c), rule, C.byref(n))
        acts = self._actions(n.value)
        self.abi.check(rc)
        return acts

    def placement_utility(self, ps: PSet, space: CandidateSpace, params: UtilityParams) -> float:
        out = C.c_double()
        self.abi.check(self.abi.placement_utility(self.s, ps.p, C.byref(space.c), C.byref(params.c),
                                                  C.byref(out)))
        return out.value
