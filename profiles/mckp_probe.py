"""oracle_mckp: exact-solver wall time on the B200 (one
subtree per thread) vs the reference's own DFS (oracle/_ref, one thread) on
random instances of growing size; both results must be identical.

  python profiles/mckp_probe.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2512_14946_b200 as pkg  # noqa: E402
from paper_2512_14946_b200 import _abi as A  # noqa: E402
from paper_2512_14946_b200.kvtier import Engine  # noqa: E402
from test_mckp import _instance  # noqa: E402


def timed(eng, inst, limit):
    ps = eng.pset(inst[0])
    t0 = time.perf_counter()
    out = eng.oracle_mckp(ps, *inst[1:], limit)
    return time.perf_counter() - t0, out


def main():
    gpu = Engine(pkg.product())
    ref = Engine(A.Abi(os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so"), "ref_", codec=False))
    timed(gpu, _instance(0, 3), 1e12)  # warm-up
    for seed, n, three, nm, hard in [(11, 6, False, 2, False), (12, 7, False, 2, False), (13, 8, False, 2, False),
                                     (14, 6, True, 2, False), (15, 7, True, 2, False), (16, 5, True, 3, False),
                                     (21, 8, False, 2, True), (22, 10, False, 2, True), (23, 12, False, 2, True),
                                     (24, 8, True, 2, True)]:
        inst = _instance(seed, n, n_methods=nm, three_tiers=three)
        if hard:  # knapsack-like: equal sizes, every context wants the fast tier uncompressed,
            # which holds half of them; near-equal utilities leave the bound loose
            a, tiers = inst[0], inst[1]
            rng = np.random.default_rng(seed)
            a.orig[:] = 4_000_000_000
            a.freq[:] = 1.0 + rng.uniform(0.0, 1e-2, a.n)
            grid = np.array([0.1, 0.4, 0.8, 1.0])
            a.qual.reshape(a.n, -1, 4)[:] = grid ** 0.3
            tiers[0].capacity_bytes = (n // 2) * 4_000_000_000
        tg, (ug, bg) = timed(gpu, inst, 1e30)
        tr, (ur, br) = timed(ref, inst, 1e30)
        same = ug == ur and all(np.array_equal(bg[f], br[f]) for f in ("tier_id", "method", "ratio"))
        cands = 2 * nm * 4 if not three else 3 * nm * 4
        print(json.dumps({"contexts": n, "candidates_per_context": cands, "knapsack_like": hard,
                          "assignment_space": float(cands) ** n, "b200_s": round(tg, 4), "reference_s": round(tr, 4),
                          "speedup": round(tr / tg, 1), "identical": bool(same)}), flush=True)


if __name__ == "__main__":
    main()
