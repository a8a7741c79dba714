"""Placement past 1,024 contexts, pinned to the reference.

The device store keeps one 32-ary tournament tree per tier; past 1,024
residents the trees are 3 levels deep (placement.cu DevStore). These cases
replay the reference's own insert_joint results at that scale, recorded by
tests/golden/make_large_golden.py from the unmodified kvtier library
(oracle/_ref, proj/src/placement.cpp:174-250):

  ws2  2 ranks x 1,000 c2 contexts (the bench's 2-GPU weak-scaling instance)
  c5   BASELINE configs[4]: 13,889 varied-length contexts, 1,000,008 candidates
  ws8  8 ranks x 1,000 c2 contexts (the 8-GPU instance), 1,728,000 candidates

The inputs are regenerated (seeded) and checked against the recorded hash.
CPU: the cached-greedy baseline (ref_insert_joint_cached) must reproduce the
recorded lists too. GPU: kvt_insert_joint, bit-exact.
"""
import os
import sys

import numpy as np
import pytest

from paper_2512_14946_b200.kvtier import Engine

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_large_golden as G  # noqa: E402

CASES = [c for c in ("ws2", "c5", "ws8") if os.path.exists(os.path.join(HERE, "golden", f"large_placement_{c}.npz"))]
SNAP_FIELDS = ("tier_index", "method", "ratio", "original_size_bytes", "frequency", "last_access")


def _load(case):
    d = np.load(os.path.join(HERE, "golden", f"large_placement_{case}.npz"))
    arrays, tiers, space, params = G.instance(case)
    assert str(d["input_sha256"]) == G.input_hash(arrays), f"{case}: workload generator drifted from the fixture"
    return d, arrays, tiers, space, params


def _check(case, d, st, ps, space, params, acts):
    assert len(acts) == len(d["actions"]), f"{case}: {len(acts)} actions vs reference {len(d['actions'])}"
    for f in ("kind", "ctx", "tier_id", "method"):
        bad = np.nonzero(acts[f] != d["actions"][f])[0]
        assert not len(bad), f"{case}: action {bad[0]} .{f} differs"
    assert np.array_equal(acts["ratio"].view(np.uint64), d["actions"]["ratio"].view(np.uint64))
    snap = st.snapshot()
    for f in SNAP_FIELDS:
        a, b = snap[f], d["snapshot"][f]
        assert np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                              b.view(np.uint64) if b.dtype == np.float64 else b), f"{case}: snapshot.{f}"
    assert np.array_equal(st.occupancy(), d["occupancy"])
    res = st.residents()
    assert [len(r) for r in res] == d["resident_counts"].tolist()
    assert np.array_equal(np.concatenate([np.asarray(r, np.int32) for r in res]), d["residents"])
    u = st.placement_utility(ps, space, params)
    assert np.float64(u).view(np.uint64) == np.float64(d["utility"]).view(np.uint64)


def test_large_fixtures_present():
    assert "ws2" in CASES, "tests/golden/large_placement_ws2.npz missing"


@pytest.mark.parametrize("case", CASES)
def test_cached_greedy_baseline_matches_reference_fixture(ref_abi, case):
    d, arrays, tiers, space, params = _load(case)
    eng = Engine(ref_abi)
    ps = eng.pset(arrays)
    st = eng.store(tiers, arrays.n, space)
    acts = st.insert_joint(ps, space, params, np.arange(arrays.n, dtype=np.int32), cached=True)
    _check(case, d, st, ps, space, params, acts)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_insert_joint_matches_reference_fixture(gpu_abi, case):
    """3-level tournament trees: the device greedy's action list, store and
    placement utility equal the reference's, bit for bit."""
    d, arrays, tiers, space, params = _load(case)
    eng = Engine(gpu_abi)
    ps = eng.pset(arrays)
    st = eng.store(tiers, arrays.n, space)
    acts = st.insert_joint(ps, space, params, np.arange(arrays.n, dtype=np.int32))
    _check(case, d, st, ps, space, params, acts)
