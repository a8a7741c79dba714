"""CUDA placement path (libkvt_b200.so) vs the reference library and the
oracle: bit-exact candidate tables, best configs, action lists, store state
and placement utility. The reference's own known answers run on the GPU
engine too (imported from test_oracle_pinned)."""
import numpy as np
import pytest

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import Engine

from cases import bench_profiles, random_instance, three_tiers
from parity import compare_runs, compare_scoring, run_inserts
from test_oracle_pinned import (test_best_config_fig2_and_ties as test_gpu_best_config_fig2_and_ties,  # noqa: F401
                                test_compressed_size_goldens as test_gpu_compressed_size_goldens,
                                test_duplicate_insert_raises as test_gpu_duplicate_insert_raises,
                                test_fig2_walkthrough as test_gpu_fig2_walkthrough,
                                test_least_drop_tie_breaking as test_gpu_least_drop_tie_breaking,
                                test_least_drop_update as test_gpu_least_drop_update,
                                test_lone_tier_recompress_and_impossible_fit as test_gpu_lone_tier,
                                test_rearrange_fixed_point_and_collapse as test_gpu_rearrange)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng(gpu_abi):
    return Engine(gpu_abi)


@pytest.mark.parametrize("seed", range(16))
def test_gpu_matches_reference_random(eng, ref_abi, seed):
    n_ctx = [6, 12, 25, 40, 80, 150][seed % 6]
    arrays, tiers, space, params = random_instance(seed + 100, n_ctx=n_ctx, n_methods=1 + seed % 3,
                                                   n_tiers=2 + seed % 2)
    er = Engine(ref_abi)
    compare_scoring(eng, er, arrays, tiers, space, params)
    order = np.random.default_rng(seed).permutation(arrays.n)
    for rule in (A.KVT_RULE_UTILITY, A.KVT_RULE_QUALITY_FIRST):
        rr = run_inserts(er, arrays, tiers, space, params, order, rule, then_rearrange=True)
        rg = run_inserts(eng, arrays, tiers, space, params, order, rule, batch=(seed % 2 == 0),
                         then_rearrange=True)
        compare_runs(rg, rr, f"seed{seed}/rule{rule}")


@pytest.mark.parametrize("seed,n_ctx", [(0, 1100), (1, 1500), (2, 1025)])
def test_gpu_matches_reference_random_deep_trees(eng, ref_abi, seed, n_ctx):
    """Past 1,024 residents the device's per-tier tournament trees grow a
    third level: seeded random instances there, live against the reference
    (insert_joint of every context, then rearrange)."""
    arrays, tiers, space, params = random_instance(seed + 4000, n_ctx=n_ctx, n_methods=3, n_tiers=3)
    er = Engine(ref_abi)
    order = np.random.default_rng(seed).permutation(arrays.n)
    rr = run_inserts(er, arrays, tiers, space, params, order, then_rearrange=True)
    rg = run_inserts(eng, arrays, tiers, space, params, order, then_rearrange=True)
    compare_runs(rg, rr, f"deep{n_ctx}")
    assert len(rr["actions"]) > 2 * n_ctx


@pytest.mark.parametrize("seed", range(4))
def test_gpu_least_drop_every_step(eng, ref_abi, seed):
    """least_drop_update on every over-full tier after every insert."""
    arrays, tiers, space, params = random_instance(seed + 500, n_ctx=30, n_methods=3, n_tiers=3)
    er = Engine(ref_abi)
    pg, pr = eng.pset(arrays), er.pset(arrays)
    sg, sr = eng.store(tiers, arrays.n, space), er.store(tiers, arrays.n, space)
    for c in np.random.default_rng(seed).permutation(arrays.n):
        ag = sg.insert_joint(pg, space, params, [c])
        ar = sr.insert_joint(pr, space, params, [c])
        assert np.array_equal(ag, ar)
    # force overflow by direct adds at ratio 1.0 on the top tier, then query
    snap = sr.snapshot()
    free = [c for c in range(arrays.n) if snap["tier_index"][c] < 0]
    assert not free
    for t in range(len(tiers) - 1):
        for s_ in (sg, sr):
            pass
    # query every finite tier (over capacity or not, the argmin is defined)
    for t in range(len(tiers)):
        try:
            ug = sg.least_drop_update(pg, space, params, t)
        except A.ValidationError:
            with pytest.raises(A.ValidationError):
                sr.least_drop_update(pr, space, params, t)
            continue
        ur = sr.least_drop_update(pr, space, params, t)
        for f in ("ctx", "kind", "tier_index", "tier_id", "method", "ratio", "size_bytes", "quality", "ttft",
                  "utility", "utility_drop", "bytes_freed"):
            assert getattr(ug, f) == getattr(ur, f), f


def test_gpu_direct_store_edits_then_resolve(eng, ref_abi):
    """StoreState::add at off-grid configs (the LRU / fixed path) then
    resolve_overflow: keep-config evictions and on-the-fly scoring."""
    arrays, tiers, space, params = random_instance(777, n_ctx=20, n_methods=2, n_tiers=3, varied_grid=False)
    er = Engine(ref_abi)
    runs = []
    for e in (eng, er):
        ps = e.pset(arrays)
        st = e.store(tiers, arrays.n, space)
        for c in range(arrays.n):
            st.add(c, 0, c % 2 if arrays.has[c, c % 2] else int(np.argmax(arrays.has[c])),
                   [1.0, 0.37, 0.55, 0.9][c % 4], int(arrays.orig[c]), c, c)
        acts = st.resolve_overflow(ps, space, params)
        runs.append((acts, st.occupancy(), st.residents(), st.placement_utility(ps, space, params)))
    (ag, og, rg, ug), (ar, or_, rr, ur) = runs
    assert np.array_equal(ag, ar) and np.array_equal(og, or_) and rg == rr and ug == ur


@pytest.mark.parametrize("n_ctx,gpu_frac,varied", [(1000, 0.10, False), (700, 0.02, True)])
def test_gpu_bench_shaped_parity(eng, ref_abi, n_ctx, gpu_frac, varied):
    """BASELINE C2/C3-shaped instances (3 tiers, tight GPU tier): full
    insert_joint sequence, bit-identical to the reference."""
    from paper_2512_14946_b200.kvtier import CandidateSpace, UtilityParams
    space = CandidateSpace(["keydiff", "knorm", "snapkv", "keydiff-q4", "knorm-q8", "snapkv-q2"],
                           [0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 1.0])
    arrays = bench_profiles(n_ctx, space, seed=n_ctx, varied=varied)
    tiers = three_tiers(int(arrays.orig.sum()), gpu_frac, 0.3)
    params = UtilityParams(alpha=1.0)
    order = np.arange(n_ctx)
    er = Engine(ref_abi)
    rr = run_inserts(er, arrays, tiers, space, params, order)
    rg = run_inserts(eng, arrays, tiers, space, params, order)
    compare_runs(rg, rr, f"bench{n_ctx}")
    assert len(rg["actions"]) > n_ctx  # the tight tier forces evictions
