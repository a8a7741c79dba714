"""Placement at scale (BASELINE configs[4]): K1 candidate
scoring + best_config and the K3 greedy (insert_joint of every context into
an empty 3-tier store) for 13,889 varied-size Llama-3.1-8B contexts =
1,000,008 (context, method, ratio, tier) candidates, on the B200, timed with
CUDA events; the action list is checked against the CPU restatement
(oracle, bit-exact). The reference's own greedy is quadratic (SURVEY §0.6:
723 s single-thread at this size); `--ref-ctx N` times it on the first N
contexts here for the record.

  python profiles/placement_probe.py [--n-ctx 13889] [--ref-ctx 1000]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_14946_b200 as pkg  # noqa: E402
from paper_2512_14946_b200 import _abi as A, workload  # noqa: E402
from paper_2512_14946_b200.kvtier import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-ctx", type=int, default=13889)
    ap.add_argument("--ref-ctx", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    W = workload.build("c5", n_ctx=args.n_ctx)
    arrays, space, params, tiers = W["arrays"], W["space"], W["params"], W["tiers"]
    ncand = arrays.n * len(space.methods) * len(space.ratios) * len(tiers)
    eng = Engine(pkg.product())
    ps = eng.pset(arrays)
    st = eng.store(tiers, arrays.n, space)
    order = np.arange(arrays.n, dtype=np.int32)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t_score, t_greedy = [], []
    for r in range(args.reps + 1):
        torch.cuda.synchronize()
        ev[0].record()
        eng.best_config(ps, tiers, space, params)  # K1 over every candidate (+ D2H of the winners)
        ev[1].record()
        st.clear()
        ev[2].record()
        acts = st.insert_joint(ps, space, params, order)
        ev[3].record()
        torch.cuda.synchronize()
        if r:
            t_score.append(ev[0].elapsed_time(ev[1]))
            t_greedy.append(ev[2].elapsed_time(ev[3]))
    orc = Engine(A.Abi(os.path.join(ROOT, "oracle", "liboracle.so"), "orc_", codec=False))
    so = orc.store(tiers, arrays.n, space)
    t0 = time.perf_counter()
    acts_o = so.insert_joint(orc.pset(arrays), space, params, order)
    t_orc = time.perf_counter() - t0
    out = {"contexts": arrays.n, "candidates": ncand, "actions": int(len(acts)),
           "score_ms": round(float(np.median(t_score)), 3), "greedy_ms": round(float(np.median(t_greedy)), 3),
           "candidates_per_s": round(ncand / (np.median(t_score) / 1e3), 0),
           "greedy_actions_per_s": round(len(acts) / (np.median(t_greedy) / 1e3), 0),
           "bit_exact_vs_oracle": bool(np.array_equal(acts, acts_o)),
           "oracle_cached_greedy_cpu_s": round(t_orc, 3)}
    if args.ref_ctx:
        ref = Engine(A.Abi(os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so"), "ref_", codec=False))
        sub = workload.build("c5", n_ctx=args.ref_ctx)
        sr = ref.store(sub["tiers"], sub["arrays"].n, space)
        t0 = time.perf_counter()
        sr.insert_joint(ref.pset(sub["arrays"]), space, params, np.arange(sub["arrays"].n))
        out["reference_greedy_cpu_s"] = {"contexts": args.ref_ctx, "seconds": round(time.perf_counter() - t0, 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
