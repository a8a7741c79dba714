"""Golden vectors produced by the reference itself (tests/golden/make_golden.py
ran the unmodified kvtier library on these exact inputs). The inputs are
rebuilt from the stored arrays (not regenerated), then the CPU oracle
(no GPU) and the CUDA engine (gpu) must reproduce every stored output bit
for bit: candidate tables, best_config under both rules, batch insert_joint
+ rearrange action lists, final snapshots, occupancy, placement utility."""
import os

import numpy as np
import pytest

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import (CandidateSpace, CompressionMethod, Engine, ProfileArrays, TierSpec,
                                          UtilityParams)

from parity import assert_same, run_inserts

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "placement_golden.npz")


def _cases():
    g = np.load(GOLD)
    for ci in range(int(g["n_cases"])):
        pre = f"c{ci}_"
        n = len(g[pre + "orig"])
        arrays = ProfileArrays([f"c{i:05d}" for i in range(n)], g[pre + "orig"], g[pre + "freq"], g[pre + "goff"],
                               g[pre + "grid"], g[pre + "qual"], g[pre + "has"].reshape(n, -1))
        tiers = [TierSpec(int(t["id"]), f"t{int(t['id'])}", None if t["cap"] < 0 else int(t["cap"]), float(t["bw"]),
                          float(t["lat"])) for t in g[pre + "tiers"]]
        space = CandidateSpace([CompressionMethod(str(m), float(o)) for m, o in
                                zip(g[pre + "methods"], g[pre + "overhead"])], [float(r) for r in g[pre + "ratios"]])
        params = UtilityParams(alpha=float(g[pre + "alpha"]))
        yield ci, g, pre, arrays, tiers, space, params


def _check(eng):
    n_checked = 0
    for ci, g, pre, arrays, tiers, space, params in _cases():
        ps = eng.pset(arrays)
        sc = eng.score_candidates(ps, tiers, space, params)
        v = g[pre + "cand_valid"].astype(bool)
        assert_same(sc["valid"], g[pre + "cand_valid"], f"case{ci}.valid")
        assert_same(sc["size"], g[pre + "cand_size"], f"case{ci}.size")
        assert_same(np.where(v, sc["quality"], 0), np.where(v, g[pre + "cand_quality"], 0), f"case{ci}.quality")
        vt = np.broadcast_to(v[:, None], sc["utility"].shape)
        for k in ("ttft", "utility"):
            assert_same(np.where(vt, sc[k], 0), np.where(vt, g[pre + "cand_" + k], 0), f"case{ci}.{k}")
        for rule in (A.KVT_RULE_UTILITY, A.KVT_RULE_QUALITY_FIRST):
            b, gb = eng.best_config(ps, tiers, space, params, rule), g[pre + f"best{rule}"]
            ok = gb["status"] == 0
            assert_same(b["status"], gb["status"], f"case{ci}.best.status")
            assert_same(b[ok], gb[ok], f"case{ci}.best{rule}")
            r = run_inserts(eng, arrays, tiers, space, params, g[pre + f"order{rule}"], rule, then_rearrange=True)
            assert (r["error"] is not None) == bool(g[pre + f"err{rule}"]), f"case{ci}: error status"
            if r["error"] is None:
                assert_same(r["actions"], g[pre + f"acts{rule}"], f"case{ci}.actions{rule}")
                assert_same(np.float64(r["utility"]), g[pre + f"util{rule}"], f"case{ci}.placement_utility")
                n_checked += len(r["actions"])
            assert_same(r["occupancy"], g[pre + f"occ{rule}"], f"case{ci}.occupancy")
            s, gs = r["snapshot"], g[pre + f"snap{rule}"]
            assert_same(s["tier_index"], gs["tier_index"], f"case{ci}.tier")
            m = gs["tier_index"] >= 0
            for f in ("method", "ratio", "original_size_bytes", "frequency", "last_access"):
                assert_same(s[f][m], gs[f][m], f"case{ci}.snapshot.{f}")
    assert n_checked > 500  # the fixtures exercise real overflow cascades


def test_oracle_reproduces_reference_golden(oracle_abi):
    _check(Engine(oracle_abi))


@pytest.mark.gpu
def test_gpu_reproduces_reference_golden(gpu_abi):
    _check(Engine(gpu_abi))
