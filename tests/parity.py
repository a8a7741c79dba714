"""Drive two ABI implementations with identical inputs and compare every
output bit-for-bit (placement is integer/index/f64 work: the bar is
bit-exact)."""
from __future__ import annotations

import numpy as np

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import Engine, ProfileArrays, StoreState


def bits(x):
    x = np.ascontiguousarray(x)
    if x.dtype == np.float64:
        return x.view(np.uint64)
    return x


def assert_same(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    if a.dtype.names:
        for f in a.dtype.names:
            if f == "pad_":
                continue
            assert_same(a[f], b[f], f"{what}.{f}")
        return
    ba, bb = bits(a), bits(b)
    bad = np.nonzero(ba != bb)
    if len(bad[0]):
        i = tuple(ix[0] for ix in bad)
        raise AssertionError(f"{what}: {len(bad[0])} mismatches, first at {i}: {a[i]!r} vs {b[i]!r}")


def compare_scoring(e1: Engine, e2: Engine, arrays: ProfileArrays, tiers, space, params):
    p1, p2 = e1.pset(arrays), e2.pset(arrays)
    s1 = e1.score_candidates(p1, tiers, space, params)
    s2 = e2.score_candidates(p2, tiers, space, params)
    assert_same(s1["valid"], s2["valid"], "valid")
    v = s1["valid"].astype(bool)
    assert_same(s1["size"], s2["size"], "size")
    assert_same(np.where(v, s1["quality"], 0), np.where(v, s2["quality"], 0), "quality")
    vt = np.broadcast_to(v[:, None], s1["ttft"].shape)
    assert_same(np.where(vt, s1["ttft"], 0), np.where(vt, s2["ttft"], 0), "ttft")
    assert_same(np.where(vt, s1["utility"], 0), np.where(vt, s2["utility"], 0), "utility")
    for rule in (A.KVT_RULE_UTILITY, A.KVT_RULE_QUALITY_FIRST):
        b1 = e1.best_config(p1, tiers, space, params, rule)
        b2 = e2.best_config(p2, tiers, space, params, rule)
        ok = b1["status"] == 0
        assert_same(b1["status"], b2["status"], "best.status")
        assert_same(b1[ok], b2[ok], f"best(rule={rule})")
    return s1


def run_inserts(eng: Engine, arrays, tiers, space, params, order, rule=A.KVT_RULE_UTILITY,
                batch=True, then_rearrange=False):
    ps = eng.pset(arrays)
    st: StoreState = eng.store(tiers, arrays.n, space)
    order = np.asarray(order, np.int32)
    freq = np.arange(len(order), dtype=np.int64) % 5
    stamp = np.arange(1, len(order) + 1, dtype=np.int64)
    err = None
    try:
        if batch:
            acts = st.insert_joint(ps, space, params, order, freq, stamp, rule)
        else:
            parts = []
            for i in range(len(order)):
                parts.append(st.insert_joint(ps, space, params, order[i:i + 1], freq[i:i + 1],
                                             stamp[i:i + 1], rule))
            acts = np.concatenate(parts) if parts else np.zeros(0, A.ACTION_DTYPE)
        if then_rearrange:
            acts = np.concatenate([acts, st.rearrange(ps, space, params, rule)])
    except A.ValidationError as e:
        err = e
        acts = None
    util = st.placement_utility(ps, space, params) if err is None else None
    return dict(actions=acts, occupancy=st.occupancy(), residents=st.residents(),
                snapshot=st.snapshot(), utility=util, error=err)


def compare_runs(r1, r2, what="run"):
    assert (r1["error"] is None) == (r2["error"] is None), f"{what}: error {r1['error']} vs {r2['error']}"
    if r1["error"] is None:
        assert_same(r1["actions"], r2["actions"], f"{what}.actions")
        assert_same(np.float64(r1["utility"]), np.float64(r2["utility"]), f"{what}.placement_utility")
    assert_same(r1["occupancy"], r2["occupancy"], f"{what}.occupancy")
    assert r1["residents"] == r2["residents"], f"{what}: per-tier arrival order differs"
    s1, s2 = r1["snapshot"], r2["snapshot"]
    for f in ("tier_index", "method", "ratio", "original_size_bytes", "frequency", "last_access"):
        m = s1["tier_index"] >= 0
        assert_same(s1[f][m], s2[f][m], f"{what}.snapshot.{f}")
