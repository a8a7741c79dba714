"""Serve loop (with f3's drift / re-profiling) against the
reference's own replay.

tests/golden/make_replay_golden.py ran the unmodified reference (scenario
loader + kvtier::replay) on its shipped scenarios and stored the expanded
inputs with the results. paper_2512_14946_b200.serve.Replayer replays the
same trace on the CPU oracle store (no GPU) and on the CUDA store (gpu):
every request record (hit / miss, serving tier, configuration, TTFT,
quality), every placement action, the final placements and the metrics
must match exactly."""
import glob
import gzip
import json
import os

import pytest

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import Engine
from paper_2512_14946_b200.serve import Replayer, Request, Scenario, replay

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "replay_*.json.gz")))


def _load(path):
    with gzip.open(path, "rt") as f:
        return json.load(f)


def _check(eng, doc):
    sc, trace = Scenario.from_doc(doc)
    res = replay(eng, sc, trace)
    ref = doc["result"]
    assert len(res.records) == len(ref["records"])
    for i, (r, g) in enumerate(zip(res.records, ref["records"])):
        assert r.hit == g["hit"], f"request {i}: hit"
        if r.hit:
            assert (r.tier, r.method, r.ratio) == (g["tier"], g["method"], g["ratio"]), f"request {i}: config"
        assert r.ttft == g["ttft"], f"request {i}: ttft {r.ttft!r} vs {g['ttft']!r}"
        assert r.quality == g["quality"], f"request {i}: quality"
    acts = [(a["kind"], a["context"], a["tier"], a["method"], a["ratio"]) for a in ref.get("actions", [])]
    assert res.actions == acts
    assert res.final_placements == ref["final_placements"]
    for k, v in ref["metrics"].items():
        assert res.metrics[k] == v, k
    assert res.reprofile_count == ref["reprofile_count"]
    assert res.profiling_windows == [(w["start"], w["duration"], w["penalty"]) for w in ref.get("profiling_windows", [])]
    return len(res.records), len(res.actions)


def test_replay_fixtures_present():
    names = {os.path.basename(p) for p in GOLD}
    assert {"replay_fig2_warm.json.gz", "replay_bimodal_cold.json.gz", "replay_drift_truth_cold.json.gz",
            "replay_drift_warm.json.gz", "replay_drift_noise.json.gz"} <= names
    # the drift fixtures re-profile and rearrange many times
    assert _load(os.path.join(os.path.dirname(GOLD[0]), "replay_drift_warm.json.gz"))["result"]["reprofile_count"] > 5


def test_mt19937_64_known_answer():
    from paper_2512_14946_b200.serve import MT19937_64
    g = MT19937_64(5489)  # C++11 [rand.predef]: the 10000th output of a default-seeded mt19937_64
    for _ in range(9999):
        g.next_u64()
    assert g.next_u64() == 9981545732273789042


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[7:-8] for p in GOLD])
def test_oracle_serve_loop_matches_reference(oracle_abi, path):
    _check(Engine(oracle_abi), _load(path))


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[7:-8] for p in GOLD])
def test_gpu_serve_loop_matches_reference(gpu_abi, path):
    n_req, _ = _check(Engine(gpu_abi), _load(path))
    assert n_req > 0


def test_serve_loop_trace_errors(oracle_abi):
    doc = _load(GOLD[0])
    sc, trace = Scenario.from_doc(doc)
    rp = Replayer(Engine(oracle_abi), sc)
    with pytest.raises(A.AbiError):
        rp.run([Request(2.0, trace[0].context), Request(1.0, trace[0].context)])  # non-monotone trace
    with pytest.raises(A.AbiError):
        rp.run([Request(5.0, "no-such-context")])
