"""Generate tests/golden/placement_golden.npz from the REFERENCE itself.

Runs the unmodified kvtier library (oracle/_ref/libkvtier_ref.so, built by
`make -C oracle` from /root/reference/proj/src) on seeded instances and
records its outputs next to the exact inputs, so the parity tests have
reference answers that do not need /root/reference (or any build of it) at
run time. Cases: tests/cases.random_instance seeds (2/3 tiers, 1-3 methods,
off-grid profile ratios, missing methods, decompression overhead), each with
a batch insert_joint + rearrange under both selection rules, plus the dense
candidate tables and best_config.

    python tests/golden/make_golden.py      # needs oracle/_ref built here
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from paper_2512_14946_b200 import _abi as A  # noqa: E402
from paper_2512_14946_b200.kvtier import Engine  # noqa: E402

from cases import random_instance  # noqa: E402
from parity import run_inserts  # noqa: E402

CASES = [dict(seed=s, n_ctx=n, n_methods=m, n_tiers=t) for s, n, m, t in
         [(11, 20, 1, 2), (12, 35, 2, 3), (13, 60, 3, 3), (14, 90, 3, 2), (15, 150, 3, 3), (16, 45, 2, 2)]]


def main():
    ref = Engine(A.Abi(os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so"), "ref_", codec=False))
    out = {}
    for ci, c in enumerate(CASES):
        arrays, tiers, space, params = random_instance(c["seed"], n_ctx=c["n_ctx"], n_methods=c["n_methods"],
                                                       n_tiers=c["n_tiers"])
        pre = f"c{ci}_"
        out[pre + "spec"] = np.array([c["seed"], c["n_ctx"], c["n_methods"], c["n_tiers"]], np.int64)
        # inputs, verbatim
        for k in ("orig", "freq", "goff", "grid", "qual", "has"):
            out[pre + k] = getattr(arrays, k)
        out[pre + "tiers"] = np.array([(t.tier_id, -1 if t.capacity_bytes is None else t.capacity_bytes,
                                        t.read_bandwidth, t.fixed_access_latency) for t in tiers],
                                      dtype=[("id", "i8"), ("cap", "i8"), ("bw", "f8"), ("lat", "f8")])
        out[pre + "methods"] = np.array([m.name for m in space.methods])
        out[pre + "overhead"] = np.array([m.decompression_overhead for m in space.methods])
        out[pre + "ratios"] = np.array(space.raw_ratios)
        out[pre + "alpha"] = np.array(params.alpha)
        # reference outputs
        ps = ref.pset(arrays)
        sc = ref.score_candidates(ps, tiers, space, params)
        for k, v in sc.items():
            out[pre + "cand_" + k] = v
        for rule in (A.KVT_RULE_UTILITY, A.KVT_RULE_QUALITY_FIRST):
            out[pre + f"best{rule}"] = ref.best_config(ps, tiers, space, params, rule)
            order = np.random.default_rng(c["seed"]).permutation(arrays.n)
            r = run_inserts(ref, arrays, tiers, space, params, order, rule, then_rearrange=True)
            out[pre + f"order{rule}"] = order
            out[pre + f"err{rule}"] = np.array(r["error"] is not None)
            if r["error"] is None:
                out[pre + f"acts{rule}"] = r["actions"]
                out[pre + f"util{rule}"] = np.array(r["utility"])
            out[pre + f"snap{rule}"] = r["snapshot"]
            out[pre + f"occ{rule}"] = r["occupancy"]
    out["n_cases"] = np.array(len(CASES))
    np.savez_compressed(os.path.join(HERE, "placement_golden.npz"), **out)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()
