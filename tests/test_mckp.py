"""oracle_mckp on the GPU against the reference's own
exact solver (oracle/_ref: kvtier::oracle_mckp through ref_oracle_mckp):
random small instances, tight capacities, ties; the total utility and every
context's chosen (tier, method, ratio) must be identical, and the two
refusals (assignment space over the limit, no feasible assignment) must
agree."""
import numpy as np
import pytest

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import (CandidateSpace, CompressionMethod, Engine, ProfileArrays, TierSpec,
                                          UtilityParams)


def _instance(seed, n, n_methods=2, grid=(0.1, 0.4, 0.8, 1.0), three_tiers=False, ties=False):
    rng = np.random.default_rng(seed)
    G = len(grid)
    orig = rng.integers(1, 9, n) * 1_000_000_000
    q = np.sort(rng.uniform(0.3, 1.0, (n, n_methods, G)), axis=2)
    if ties:
        q = np.round(q, 1)
    q[:, :, -1] = 1.0
    arrays = ProfileArrays.uniform_grid([f"ctx{i}" for i in range(n)], orig, rng.uniform(0.5, 3.0, n), grid, q)
    total = int(orig.sum())
    tiers = [TierSpec(0, "fast", int(total * rng.uniform(0.15, 0.5)), 20e9, 1e-4)]
    if three_tiers:
        tiers.append(TierSpec(1, "mid", int(total * rng.uniform(0.1, 0.4)), 5e9, 1e-3))
    tiers.append(TierSpec(len(tiers), "slow", None, 1e9, 1e-2))
    space = CandidateSpace([CompressionMethod(m, o) for m, o in zip(["keydiff", "knorm", "snapkv"][:n_methods],
                                                                      [0.0, 1e-12, 2e-12])], list(grid))
    return arrays, tiers, space, UtilityParams(alpha=float(rng.uniform(0.5, 5.0)))


def _solve(eng, arrays, tiers, space, params, limit=1e7):
    return eng.oracle_mckp(eng.pset(arrays), tiers, space, params, limit)


CASES = [(s, n, tt, ties) for s, (n, tt, ties) in enumerate(
    [(1, False, False), (2, False, False), (3, False, True), (4, False, False), (4, True, False), (5, False, True),
     (5, True, False), (6, False, False), (3, True, True), (6, False, True)])]


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n,three,ties", CASES)
def test_gpu_mckp_matches_reference(gpu_abi, ref_abi, seed, n, three, ties):
    inst = _instance(seed, n, three_tiers=three, ties=ties)
    tg, bg = _solve(Engine(gpu_abi), *inst, limit=1e9)
    tr, br = _solve(Engine(ref_abi), *inst, limit=1e9)
    assert tg == tr
    for f in ("tier_id", "method", "ratio", "size_bytes", "quality", "ttft", "utility"):
        assert np.array_equal(bg[f], br[f]), f


@pytest.mark.gpu
def test_gpu_mckp_refusals_match_reference(gpu_abi, ref_abi):
    inst = _instance(99, 6, n_methods=3, grid=(0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 1.0), three_tiers=True)
    for abi in (gpu_abi, ref_abi):  # 72^6 assignments > 1e7
        with pytest.raises(A.ValidationError):
            _solve(Engine(abi), *inst)
    arrays, tiers, space, params = _instance(5, 3)
    finite = [TierSpec(0, "only", 1, 1e9, 0.0)]  # nothing fits one byte
    for abi in (gpu_abi, ref_abi):
        with pytest.raises(A.ValidationError):
            _solve(Engine(abi), arrays, finite, space, params)


def test_reference_mckp_glue(ref_abi):
    total, best = _solve(Engine(ref_abi), *_instance(1, 3))
    assert np.isfinite(total) and len(best) == 3 and (best["status"] == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("n,free", [(40, 5), (200, 6)])
def test_gpu_mckp_many_forced_contexts(gpu_abi, ref_abi, n, free):
    """More than 24 contexts: the reference refuses only when the product of
    candidate counts exceeds max_assignments, so an instance of mostly
    single-candidate contexts (profile grid {1.0} under a {0.5, 0.75, 1.0}
    space: one scorable ratio) is solved exactly; one finite tier keeps the
    capacity test live at every level."""
    rng = np.random.default_rng(n)
    grid_free = [0.5, 0.75, 1.0]
    ids, orig, freq, goff, gridv, qual = [], [], [], [0], [], []
    for i in range(n):
        g = grid_free if i % (n // free) == 0 else [1.0]
        ids.append(f"c{i:04d}")
        orig.append(int(rng.integers(1, 9)) * 1_000_000_000)
        freq.append(float(rng.uniform(0.5, 3.0)))
        gridv += g
        qual += sorted(rng.uniform(0.5, 1.0, len(g)).tolist())[:-1] + [1.0]
        goff.append(len(gridv))
    arrays = ProfileArrays(ids, np.array(orig), np.array(freq), np.array(goff), np.array(gridv), np.array(qual),
                           np.ones((n, 1), np.uint8))
    free_bytes = sum(o for i, o in enumerate(orig) if i % (n // free) == 0)
    tiers = [TierSpec(0, "only", int(sum(orig) - 0.3 * free_bytes), 20e9, 1e-4)]  # the free contexts must shrink
    space = CandidateSpace([CompressionMethod("keydiff", 0.0)], grid_free)
    params = UtilityParams(alpha=2.0)
    tg, bg = _solve(Engine(gpu_abi), arrays, tiers, space, params)
    tr, br = _solve(Engine(ref_abi), arrays, tiers, space, params)
    assert tg == tr
    for f in ("tier_id", "method", "ratio", "size_bytes", "utility"):
        assert np.array_equal(bg[f], br[f]), f
    assert (br["ratio"] < 1.0).any()  # the capacity forces some compression
