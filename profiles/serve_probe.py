"""Serve-loop throughput: requests/s of
paper_2512_14946_b200.serve.Replayer on the B200 store vs the reference's
own replay (oracle/_ref/libkvtier_ref.so: scenario loader + kvtier::replay,
single thread) on the same inline scenario: N contexts with generated
profiles over a 3-tier hierarchy, a cold store, and a Zipf-skewed trace, so
every context's first request is a miss (insert_joint) and the rest are
hits. Parity of the two runs is checked on the records.

  python profiles/serve_probe.py [--n-ctx 1000] [--requests 20000]
"""
from __future__ import annotations

import argparse
import ctypes as C
import gzip
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2512_14946_b200 as pkg  # noqa: E402
from paper_2512_14946_b200.kvtier import Engine  # noqa: E402
from paper_2512_14946_b200.serve import Scenario, replay  # noqa: E402


def make_scenario(n_ctx: int, n_req: int, seed: int = 3) -> dict:
    rng = np.random.default_rng(seed)
    grid = [0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 1.0]
    methods = ["keydiff", "knorm", "snapkv"]
    profiles = []
    for i in range(n_ctx):
        size = int(rng.integers(2, 20)) * 250_000_000
        sens = rng.uniform(0.02, 0.6, 3)
        prof = {"context_id": f"ctx{i:06d}", "size_bytes": size, "frequency": float(rng.uniform(0.5, 4.0)),
                "grid": grid, "methods": {}}
        for m, s in zip(methods, sens):
            prof["methods"][m] = {("%g" % r): float(np.clip(1.0 - s * ((1.0 - r) / 0.1) ** 1.3, 0.0, 1.0))
                                  for r in grid}
        profiles.append(prof)
    total = sum(p["size_bytes"] for p in profiles)
    zipf = rng.zipf(1.3, n_req) % n_ctx
    trace = [{"t": float(t), "context_id": f"ctx{int(c):06d}", "n_new_tokens": int(rng.integers(16, 512))}
             for t, c in zip(np.cumsum(rng.exponential(0.01, n_req)), zipf)]
    return {"seed": seed, "alpha": 3.0, "policy": "joint", "warm_start": False,
            "tiers": [{"name": "gpu", "capacity_gb": total * 0.08 / 1e9, "read_bandwidth_gbps": 1000},
                      {"name": "cpu", "capacity_gb": total * 0.3 / 1e9, "read_bandwidth_gbps": 50},
                      {"name": "ssd", "read_bandwidth_gbps": 5}],
            "profiles": {"inline": profiles}, "trace": {"inline": trace}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-ctx", type=int, default=1000)
    ap.add_argument("--requests", type=int, default=20000)
    args = ap.parse_args()
    ref = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so"))
    ref.ref_replay_dump.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), C.c_int32]
    ref.ref_last_error.restype = C.c_char_p
    with tempfile.TemporaryDirectory() as d:
        scen = os.path.join(d, "s.json")
        json.dump(make_scenario(args.n_ctx, args.requests), open(scen, "w"))
        out = os.path.join(d, "r.json")
        t0 = time.perf_counter()
        rc = ref.ref_replay_dump(scen.encode(), out.encode(), None, 0)
        t_ref = time.perf_counter() - t0  # loader + replay + JSON write: an upper bound on its replay
        if rc:
            raise RuntimeError(ref.ref_last_error().decode())
        doc = json.load(open(out))
    sc, trace = Scenario.from_doc(doc)
    eng = Engine(pkg.product())
    replay(eng, sc, trace[:200])  # warm the CUDA context and code paths
    t0 = time.perf_counter()
    res = replay(eng, sc, trace)
    t_gpu = time.perf_counter() - t0
    g = doc["result"]["records"]
    exact = all(r.hit == x["hit"] and r.ttft == x["ttft"] and r.quality == x["quality"] for r, x in zip(res.records, g))
    exact = exact and len(res.actions) == len(doc["result"]["actions"])
    n = len(trace)
    misses = sum(1 for r in res.records if not r.hit)
    print(json.dumps({"contexts": args.n_ctx, "requests": n, "misses": misses, "actions": len(res.actions),
                      "b200_serve_s": round(t_gpu, 3), "b200_requests_per_s": round(n / t_gpu, 1),
                      "reference_replay_s_upper": round(t_ref, 3), "reference_requests_per_s_lower": round(n / t_ref, 1),
                      "bit_exact_vs_reference": bool(exact)}), flush=True)


if __name__ == "__main__":
    main()
