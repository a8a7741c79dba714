"""Scenario ingestion: paper_2512_14946_b200.scenario
reads the reference's own scenario files (oracle/_ref/scenarios, copied from
the reference by oracle/Makefile; the same files the reference's acceptance
gate reads) and must produce exactly the scenario the reference's loader
produced for the golden replays (tests/golden/replay_*.json.gz): tiers,
params, methods and grid, every generated profile (sizes, frequencies,
quality tables), truth curves, context order, every generated request, the
drift settings and flags. The loaded scenario then replays bit-exactly on
the oracle store."""
import glob
import gzip
import json
import os

import pytest

from paper_2512_14946_b200.kvtier import Engine
from paper_2512_14946_b200.scenario import apply_override, load_scenario_file
from paper_2512_14946_b200.serve import replay

HERE = os.path.dirname(os.path.abspath(__file__))
SCEN = os.path.join(HERE, "..", "oracle", "_ref", "scenarios")
GOLD = sorted(glob.glob(os.path.join(HERE, "golden", "replay_*.json.gz")))


def _gold(path):
    with gzip.open(path, "rt") as f:
        return json.load(f)


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[7:-8] for p in GOLD])
def test_loader_matches_reference_loader(path):
    g = _gold(path)
    src = os.path.join(SCEN, g["case"]["scenario"])
    if not os.path.exists(src):
        pytest.skip("oracle/_ref/scenarios not built here")
    sc, trace, policy = load_scenario_file(src, g["case"]["overrides"])
    assert policy == g["policy"]
    assert [(t.tier_id, t.name, t.capacity_bytes, t.read_bandwidth, t.fixed_access_latency) for t in sc.tiers] == \
        [(t["tier_id"], t["name"], t["capacity_bytes"], t["read_bandwidth"], t["fixed_access_latency"])
         for t in g["tiers"]]
    p = sc.params
    assert (p.alpha, p.prefill_a, p.prefill_b, p.bytes_per_token) == tuple(
        g["params"][k] for k in ("alpha", "prefill_a", "prefill_b", "bytes_per_token"))
    assert [(m.name, m.decompression_overhead) for m in sc.space.methods] == \
        [(m["name"], m["decompression_overhead"]) for m in g["methods"]]
    assert sc.space.ratios == g["ratios"]
    mine = {q.context: q for q in sc.profiles}
    assert sorted(mine) == [q["context"] for q in g["profiles"]]
    for q in g["profiles"]:
        m = mine[q["context"]]
        assert (m.original_size_bytes, m.frequency, m.ratio_grid) == (q["size"], q["frequency"], q["grid"]), q["context"]
        assert m.quality_table == q.get("quality", {}), q["context"]
    assert {c: {m: list(v) for m, v in t.items()} for c, t in sc.truth.items()} == (g.get("truth") or {})
    assert sc.order == g["order"]
    assert [(r.t, r.context, r.n_new_tokens) for r in trace] == \
        [(r["t"], r["context"], r["n_new_tokens"]) for r in g["trace"]]
    assert (sc.warm_start, sc.miss_store_bottom, sc.drift, sc.seed) == \
        (g["warm_start"], g["miss_store_bottom"], g["drift"], g["seed"])
    if sc.drift:
        assert sc.drift_config == g["drift_config"]


def test_loaded_scenario_replays_like_the_reference(oracle_abi):
    g = _gold(os.path.join(HERE, "golden", "replay_bimodal_cold.json.gz"))
    src = os.path.join(SCEN, "bimodal.json")
    if not os.path.exists(src):
        pytest.skip("oracle/_ref/scenarios not built here")
    sc, trace, _ = load_scenario_file(src, ["warm_start=false"])
    res = replay(Engine(oracle_abi), sc, trace)
    assert [(r.hit, r.ttft, r.quality) for r in res.records] == \
        [(r["hit"], r["ttft"], r["quality"]) for r in g["result"]["records"]]


def test_overrides():
    doc = {"tiers": [{"capacity_gb": 8}, {"name": "slow"}], "drift": None}
    apply_override(doc, "tiers.0.capacity_gb=12")
    apply_override(doc, "drift.threshold=0.25")
    apply_override(doc, "policy=lru")
    assert doc["tiers"][0]["capacity_gb"] == 12 and doc["drift"] == {"threshold": 0.25} and doc["policy"] == "lru"
