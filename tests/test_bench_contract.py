"""bench.py's JSON line keeps the driver's contract: the keys the task
names, in both arms (`--impl reference` on the CPU, the B200 arm on a GPU),
on a small workload so the run takes seconds."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # exactly one JSON line on stdout
    return json.loads(lines[0])


def _common(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert "workload" in d["config"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    assert d["cpu_baseline"]["kind"] in ("reference", "port")


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--n-ctx", "16", "--steps", "1", "--warmup", "3", "--cpu-seconds", "1"], 600)
    _common(d)
    assert d["impl"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] == d["cpu_baseline"]["value"]


@pytest.mark.gpu
def test_b200_arm_contract():
    d = _run(["--n-ctx", "16", "--steps", "1", "--warmup", "3", "--no-n1", "--tiered-steps", "0",
              "--cpu-seconds", "1"], 1200)
    _common(d)
    assert d["n_gpus"] == 1 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] <= 1.0 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3
    c = d["clocks"]
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in c, k


@pytest.mark.gpu
def test_b200_lane_trace_diagnostic():
    """--lane-trace adds one traced step and reports the cross-stream waits on
    stderr; stdout keeps exactly one JSON line."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--n-ctx", "16", "--steps", "1", "--warmup",
                        "3", "--no-n1", "--tiered-steps", "0", "--no-cpu-baseline", "--lane-trace"],
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert len([l for l in r.stdout.strip().splitlines() if l.startswith("{")]) == 1
    tr = [json.loads(l)["lane_trace"] for l in r.stderr.splitlines() if l.startswith('{"lane_trace"')]
    assert len(tr) == 1
    t = tr[0]
    assert len(t["lane_end_ms"]) == len(t["pack_lane_wait_on_scores_ms"]) >= 2
    assert all(x >= 0 for x in t["pack_lane_wait_on_scores_ms"]) and t["score_lane_scoring_ms"] >= 0
