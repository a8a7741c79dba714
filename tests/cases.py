"""Shared parity cases: the reference's own fixtures (proj/tests/*.cpp) and
seeded random instances, expressed as ProfileArrays + tiers + space."""
from __future__ import annotations

import numpy as np

from paper_2512_14946_b200.kvtier import (CandidateSpace, CompressionMethod, ContextProfile,
                                          ProfileArrays, TierSpec, UtilityParams)


def two_tiers(fast_cap=8_000_000_000):  # proj/tests/test_placement.cpp:22-33
    return [TierSpec(0, "fast", fast_cap, 20e9, 0.0), TierSpec(1, "slow", None, 2e9, 0.0)]


def flat_profile(cid, nbytes, frequency=1.0):  # proj/tests/test_placement.cpp:35-44
    return ContextProfile(cid, nbytes, frequency, [0.05, 1.0], {"keydiff": [1.0, 1.0]})


def worked_profiles():  # Fig. 2 pair, proj/tests/test_placement.cpp:48-59
    c2 = ContextProfile("ctx2", 8_000_000_000, 1.0, [0.05, 0.9, 1.0], {"keydiff": [0.5, 0.5, 1.0]})
    return [flat_profile("ctx1", 4_000_000_000), c2]


def three_tiers(total_bytes, gpu_frac=0.10, cpu_frac=0.30):
    """SURVEY §3 hierarchy: gpu 10% @8e12, cpu 30% @5e10, ssd unlimited @6e9 + 1e-4 s."""
    return [TierSpec(0, "gpu", int(total_bytes * gpu_frac), 8e12, 0.0),
            TierSpec(1, "cpu", int(total_bytes * cpu_frac), 5e10, 0.0),
            TierSpec(2, "ssd", None, 6e9, 1e-4)]


def synth_quality(s, k, r):  # proj/src/quality.cpp:115-127
    drop = s * ((1.0 - r) / 0.1) ** k
    return min(max(1.0 - drop, 0.0), 1.0)


def random_instance(seed, n_ctx=40, n_methods=3, ratios=None, n_tiers=3, gpu_frac=None,
                    varied_grid=True, off_profile=True, overhead=True, sizes="varied"):
    """A seeded instance in the spirit of gen_oracle_instance
    (proj/src/workload.cpp:627-694) and the randomized joint workloads
    (proj/tests/test_placement.cpp:674-739), widened to 3 tiers, several
    methods, per-context grids that differ from the space grid (so off-grid
    ratios interpolate) and methods missing from some profiles."""
    rng = np.random.default_rng(seed)
    names = ["keydiff", "knorm", "snapkv", "keydiff-q8", "knorm-q4", "snapkv-q2"][:n_methods]
    methods = [CompressionMethod(nm, (1e-11 if (overhead and rng.random() < 0.3) else 0.0)) for nm in names]
    if ratios is None:
        ratios = [0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 1.0]
    space = CandidateSpace(methods, ratios)
    profs = []
    total = 0
    for i in range(n_ctx):
        if sizes == "fixed":
            nbytes = 1 << 30
        else:
            nbytes = int(1e8) * int(1 + rng.integers(0, 100))
        total += nbytes
        if varied_grid and rng.random() < 0.5:
            pool = [0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
            k = int(rng.integers(1, 6))
            grid = sorted(rng.choice(pool, size=k, replace=False).tolist()) + [1.0]
        else:
            grid = sorted(set(ratios) | {1.0})
        table = {}
        for nm in names:
            if off_profile and rng.random() < 0.1 and len(table) > 0:
                continue  # method not profiled for this context
            s = rng.random()
            k = float(np.exp(rng.uniform(np.log(0.5), np.log(2.0))))
            table[nm] = [synth_quality(s, k, r) for r in grid]
        if not table:
            table[names[0]] = [1.0] * len(grid)
        profs.append(ContextProfile(f"c{i}", nbytes, float(rng.uniform(0.1, 3.0)), grid, table))
    if n_tiers == 2:
        frac = rng.uniform(0.15, 0.8) if gpu_frac is None else gpu_frac
        tiers = [TierSpec(0, "fast", int(total * frac), 20e9, float(rng.uniform(0, 0.02))),
                 TierSpec(1, "slow", None, 2e9, float(rng.uniform(0, 0.05)))]
    else:
        frac = rng.uniform(0.03, 0.3) if gpu_frac is None else gpu_frac
        tiers = three_tiers(total, frac, rng.uniform(0.1, 0.4))
    params = UtilityParams(alpha=float(rng.uniform(0.2, 3.0)))
    arrays = ProfileArrays.from_profiles(profs, space)
    return arrays, tiers, space, params


def bench_profiles(n_ctx, space, seed=7, tokens=8192, bytes_per_token=131072, varied=False):
    """Synthetic profiles for the bench configs: one shared
    grid (the space grid), sensitivity-anchored curves per method
    (synth_quality), Zipf-shaped frequencies (assign_zipf_frequencies,
    proj/src/workload.cpp:236-245, rate 4, exponent 1)."""
    rng = np.random.default_rng(seed)
    M = len(space.methods)
    grid = sorted(space.ratios)
    if varied:
        orig = (rng.integers(1024, 2 * tokens, size=n_ctx) * bytes_per_token).astype(np.int64)
    else:
        orig = np.full(n_ctx, tokens * bytes_per_token, np.int64)
    s = rng.uniform(0.02, 0.8, size=(n_ctx, M))
    # quantised variants lose a little more quality
    for m, meth in enumerate(space.methods):
        if "-q" in meth.name:
            b = int(meth.name.split("-q")[1])
            s[:, m] = np.minimum(1.0, s[:, m] * (1.0 + 0.5 * (8 - b) / 8))
    g = np.asarray(grid)
    q = np.clip(1.0 - s[:, :, None] * ((1.0 - g[None, None, :]) / 0.1), 0.0, 1.0)
    q[:, :, -1] = 1.0
    ranks = rng.permutation(n_ctx)
    w = 1.0 / (ranks + 1.0)
    freq = 4.0 * w / w.sum()
    ids = [f"ctx-{i:07d}" for i in range(n_ctx)]
    return ProfileArrays.uniform_grid(ids, orig, freq, grid, q)
