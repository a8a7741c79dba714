"""Pins the CPU oracle (oracle/orc_placement.c) before it is trusted:
(1) the reference's own known answers (proj/tests/test_utility.cpp,
test_placement.cpp, test_core.cpp), asserted on both the oracle and the
reference library compiled from /root/reference (oracle/_ref); (2) bit
equality oracle == reference on seeded random instances."""
import numpy as np
import pytest

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import (CandidateSpace, CompressionMethod, ContextProfile, Engine,
                                          ProfileArrays, TierSpec, UtilityParams, ValidationError)

from cases import flat_profile, random_instance, two_tiers, worked_profiles
from parity import compare_runs, compare_scoring, run_inserts


@pytest.fixture(params=["orc", "ref"])
def eng(request, oracle_abi, ref_abi):
    return Engine(oracle_abi if request.param == "orc" else ref_abi)


def _arr(profs, space):
    return ProfileArrays.from_profiles(profs, space)


def test_compressed_size_goldens(eng):
    # proj/tests/test_core.cpp:12-20, through the candidate size table
    cases = [(4_000_000_000, 0.05, 200_000_000), (8_000_000_000, 1.0, 8_000_000_000),
             (1000, 0.5, 500), (3, 0.5, 2), (5, 0.25, 1), (10, 0.01, 1), (1, 0.000001, 1)]
    for orig, ratio, want in cases:
        space = CandidateSpace(["keydiff"], [ratio])
        arr = _arr([ContextProfile("c", orig, 1.0, [ratio, 1.0] if ratio < 1 else [1.0],
                                   {"keydiff": [1.0, 1.0] if ratio < 1 else [1.0]})], space)
        s = eng.score_candidates(eng.pset(arr), two_tiers(), space, UtilityParams())
        assert s["size"][0, 0] == want, (orig, ratio)


def test_score_candidate_fig2(eng):
    # proj/tests/test_utility.cpp:152-173
    space = CandidateSpace.default_space()
    arr = _arr([flat_profile("ctx1", 4_000_000_000)], space)
    s = eng.score_candidates(eng.pset(arr), two_tiers(), space, UtilityParams())
    r = space.ratios.index(0.05)
    assert s["size"][0, r] == 200_000_000
    assert s["quality"][0, 0, r] == 1.0
    assert abs(s["ttft"][0, 0, 0, r] - 0.01) < 1e-14
    assert abs(s["utility"][0, 0, 0, r] - 0.99) < 1e-14
    assert abs(s["utility"][0, 1, 0, r] - 0.9) < 1e-14
    assert s["valid"][0].sum() == 8  # only keydiff is profiled


def test_best_config_fig2_and_ties(eng):
    # proj/tests/test_utility.cpp:175-223
    space = CandidateSpace.default_space()
    b = eng.best_config(eng.pset(_arr([flat_profile("ctx1", 4_000_000_000)], space)), two_tiers(),
                        space, UtilityParams())[0]
    assert (b["tier_id"], b["method"], b["ratio"]) == (0, 0, 0.05)
    assert abs(b["utility"] - 0.99) < 1e-14
    # identical methods fall back to name order
    p = flat_profile("ctx1", 4_000_000_000)
    p.quality_table = {m: [1.0, 1.0] for m in ("snapkv", "knorm", "keydiff")}
    sp2 = CandidateSpace(["snapkv", "knorm", "keydiff"], space.ratios)
    b = eng.best_config(eng.pset(_arr([p], sp2)), two_tiers(), sp2, UtilityParams())[0]
    assert sp2.method_names[b["method"]] == "keydiff"
    # flat quality prefers the larger ratio at equal utility (1-byte context)
    p = ContextProfile("c", 1, 1.0, [0.05, 1.0], {"keydiff": [1.0, 1.0]})
    b = eng.best_config(eng.pset(_arr([p], space)), two_tiers()[:1], space, UtilityParams())[0]
    assert b["ratio"] == 1.0
    # quality-first (proj/tests/test_utility.cpp:323-340)
    p = ContextProfile("c", 8_000_000_000, 1.0, [0.05, 1.0], {"keydiff": [0.9, 1.0]})
    sp3 = CandidateSpace(["keydiff", "knorm", "snapkv"], [0.05, 1.0])
    ps = eng.pset(_arr([p], sp3))
    assert eng.best_config(ps, two_tiers(), sp3, UtilityParams(), A.KVT_RULE_UTILITY)[0]["ratio"] == 0.05
    q = eng.best_config(ps, two_tiers(), sp3, UtilityParams(), A.KVT_RULE_QUALITY_FIRST)[0]
    assert q["ratio"] == 1.0 and q["quality"] == 1.0
    # unscorable everywhere reports status 1 (ValidationError in the reference)
    p = ContextProfile("c", 1000, 1.0, [0.5, 1.0], {"exotic": [0.9, 1.0]})
    b = eng.best_config(eng.pset(_arr([p], space)), two_tiers(), space, UtilityParams())[0]
    assert b["status"] == 1


def test_fig2_walkthrough(eng):
    # proj/tests/test_placement.cpp:147-183
    space = CandidateSpace.default_space()
    arr = _arr(worked_profiles(), space)
    ps = eng.pset(arr)
    st = eng.store(two_tiers(), arr.n, space)
    a1 = st.insert_joint(ps, space, UtilityParams(), [0], [0], [1])
    assert len(a1) == 1 and a1[0]["kind"] == A.KVT_INSERT and a1[0]["tier_id"] == 0
    assert a1[0]["ratio"] == 0.05
    a2 = st.insert_joint(ps, space, UtilityParams(), [1], [0], [2])
    assert [(a["kind"], a["ctx"], a["tier_id"], a["ratio"]) for a in a2] == [
        (A.KVT_INSERT, 1, 0, 1.0), (A.KVT_EVICT, 0, 1, 0.05)]
    assert st.occupancy().tolist() == [8_000_000_000, 200_000_000]
    assert st.residents() == [[1], [0]]
    assert abs(st.placement_utility(ps, space, UtilityParams()) - 1.5) < 1e-12


def test_least_drop_update(eng):
    # proj/tests/test_placement.cpp:185-217
    profs = worked_profiles()
    profs[1].ratio_grid = [0.05, 0.5, 1.0]
    profs[1].quality_table["keydiff"] = [0.5, 0.5, 1.0]
    space = CandidateSpace(["keydiff", "knorm", "snapkv"], [0.05, 0.5, 1.0])
    arr = _arr(profs, space)
    ps = eng.pset(arr)
    st = eng.store(two_tiers(), arr.n, space)
    st.add(0, 0, 0, 0.05, 4_000_000_000)
    st.add(1, 0, 0, 1.0, 8_000_000_000)
    u = st.least_drop_update(ps, space, UtilityParams(), 0)
    assert (u.ctx, u.kind, u.tier_index, u.ratio) == (0, A.KVT_EVICT, 1, 0.05)
    assert abs(u.utility_drop - 0.09) < 1e-9 and u.bytes_freed == 200_000_000


def test_least_drop_tie_breaking(eng):
    # proj/tests/test_placement.cpp:219-276
    tiers = [TierSpec(0, "t0", 1_000_000_000, 2e9), TierSpec(1, "t1", None, 2e9)]
    space = CandidateSpace(["keydiff", "knorm", "snapkv"], [1.0])
    profs = [ContextProfile("big", 2_000_000_000, 1.0, [1.0], {"keydiff": [1.0]}),
             ContextProfile("small", 1_000_000_000, 1.0, [1.0], {"keydiff": [1.0]})]
    arr = _arr(profs, space)
    st = eng.store(tiers, arr.n, space)
    for cid in ("small", "big"):
        i = arr.index[cid]
        st.add(i, 0, 0, 1.0, int(arr.orig[i]))
    u = st.least_drop_update(eng.pset(arr), space, UtilityParams(), 0)
    assert u.utility_drop == 0.0 and arr.ids[u.ctx] == "big" and u.bytes_freed == 2_000_000_000
    profs = [ContextProfile(c, 1_500_000_000, 1.0, [1.0], {"keydiff": [1.0]}) for c in ("b", "a", "c")]
    arr = _arr(profs, space)
    st = eng.store(tiers, arr.n, space)
    for cid in ("b", "a", "c"):
        i = arr.index[cid]
        st.add(i, 0, 0, 1.0, int(arr.orig[i]))
    u = st.least_drop_update(eng.pset(arr), space, UtilityParams(), 0)
    assert arr.ids[u.ctx] == "a"


def test_lone_tier_recompress_and_impossible_fit(eng):
    # proj/tests/test_placement.cpp:278-318
    space = CandidateSpace(["keydiff", "knorm", "snapkv"], [0.05, 0.5, 1.0])
    p = ContextProfile("c", 1_000_000_000, 1.0, [0.05, 0.5, 1.0], {"keydiff": [0.5, 0.9, 1.0]})
    arr = _arr([p], space)
    st = eng.store([TierSpec(0, "only", 600_000_000, 20e9)], 1, space)
    acts = st.insert_joint(eng.pset(arr), space, UtilityParams(), [0], [0], [1])
    assert [(a["kind"], a["ratio"]) for a in acts] == [(A.KVT_INSERT, 1.0), (A.KVT_RECOMPRESS, 0.5)]
    assert st.occupancy().tolist() == [500_000_000]
    tiny = eng.store([TierSpec(0, "tiny", 40_000_000, 20e9)], 1, space)
    with pytest.raises(ValidationError):
        tiny.insert_joint(eng.pset(arr), space, UtilityParams(), [0], [0], [1])


def test_rearrange_fixed_point_and_collapse(eng):
    # proj/tests/test_placement.cpp:769-817
    space = CandidateSpace.default_space()
    profs = worked_profiles()
    arr = _arr(profs, space)
    ps = eng.pset(arr)
    st = eng.store(two_tiers(), arr.n, space)
    st.insert_joint(ps, space, UtilityParams(), [0, 1], [0, 0], [1, 2])
    before = st.placement_utility(ps, space, UtilityParams())
    st.rearrange(ps, space, UtilityParams())
    assert abs(st.placement_utility(ps, space, UtilityParams()) - before) < 1e-12
    assert st.residents() == [[1], [0]]
    profs[1].quality_table["keydiff"] = [1.0, 1.0, 1.0]
    ps2 = eng.pset(_arr(profs, space))
    st.rearrange(ps2, space, UtilityParams())
    snap = st.snapshot()
    assert snap["tier_index"].tolist() == [0, 0] and snap["ratio"][1] == 0.05
    st.touch(0, 77)
    st.rearrange(ps2, space, UtilityParams())
    assert st.snapshot()["last_access"][0] == 77


def test_duplicate_insert_raises(eng):
    space = CandidateSpace.default_space()
    arr = _arr(worked_profiles(), space)
    st = eng.store(two_tiers(), arr.n, space)
    ps = eng.pset(arr)
    st.insert_joint(ps, space, UtilityParams(), [0])
    with pytest.raises(ValidationError):
        st.insert_joint(ps, space, UtilityParams(), [0])


@pytest.mark.parametrize("seed", range(12))
def test_oracle_matches_reference_random(oracle_abi, ref_abi, seed):
    n_ctx = [6, 12, 25, 40][seed % 4]
    arrays, tiers, space, params = random_instance(seed, n_ctx=n_ctx, n_methods=1 + seed % 3,
                                                   n_tiers=2 + seed % 2)
    eo, er = Engine(oracle_abi), Engine(ref_abi)
    compare_scoring(eo, er, arrays, tiers, space, params)
    order = np.random.default_rng(seed).permutation(arrays.n)
    for rule in (A.KVT_RULE_UTILITY, A.KVT_RULE_QUALITY_FIRST):
        ro = run_inserts(eo, arrays, tiers, space, params, order, rule, then_rearrange=True)
        rr = run_inserts(er, arrays, tiers, space, params, order, rule, then_rearrange=True)
        compare_runs(ro, rr, f"seed{seed}/rule{rule}")


@pytest.mark.parametrize("seed", range(6))
def test_cached_greedy_baseline_equals_reference(ref_abi, seed):
    """ref_insert_joint_cached (the single-core CPU baseline of the cached
    per-resident best update, on the reference's own scoring
    functions) reproduces the reference's insert_joint exactly: actions,
    store, placement utility, errors."""
    from cases import random_instance
    from parity import compare_runs
    eng = Engine(ref_abi)
    arrays, tiers, space, params = random_instance(seed + 900, n_ctx=[40, 80, 150, 300, 30, 60][seed],
                                                   n_methods=1 + seed % 3, n_tiers=2 + seed % 2)
    order = np.random.default_rng(seed).permutation(arrays.n)
    runs = []
    for cached in (False, True):
        ps = eng.pset(arrays)
        st = eng.store(tiers, arrays.n, space)
        err = None
        try:
            acts = st.insert_joint(ps, space, params, order, cached=cached)
        except A.ValidationError as e:
            acts, err = None, str(e)
        runs.append(dict(actions=acts, occupancy=st.occupancy(), residents=st.residents(), snapshot=st.snapshot(),
                         utility=None if err else st.placement_utility(ps, space, params), error=err))
    compare_runs(runs[1], runs[0], f"seed{seed}")
    assert runs[1]["error"] == runs[0]["error"]
