"""Generate tests/golden/large_placement_<case>.npz from the REFERENCE itself:
placement instances past 1,024 contexts, where the device store's per-tier
tournament trees are 3 levels deep (kvt_b200 placement.cu DevStore).

Runs the unmodified kvtier greedy (oracle/_ref/libkvtier_ref.so, built by
`make -C oracle` from /root/reference/proj/src) — insert_joint over every
context in arrival order, proj/src/placement.cpp:225-250 — and records the
full action list, the final store snapshot, the per-tier occupancy and
placement_utility (placement.cpp:285-298). The inputs are not stored: they
are regenerated bit-identically by paper_2512_14946_b200.workload (seeded
numpy), and a hash of them is stored so a drifted generator fails loudly.

Cases
  c5   BASELINE configs[4]: 13,889 varied-length Llama-3.1-8B contexts x
       3 methods x 8 ratios x 3 tiers = 1,000,008 candidates (~12 min here)
  ws8  the bench's 8-rank weak-scaling instance: 8 x 1,000 c2 contexts
       (seeds 7..14, rank-major ids, distributed.merge_rank_profiles),
       9 methods x 8 ratios x 3 tiers = 1,728,000 candidates
  ws2  the same at 2 ranks (2,000 contexts)

    python tests/golden/make_large_golden.py [case ...]   # needs oracle/_ref
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2512_14946_b200 import _abi as A  # noqa: E402
from paper_2512_14946_b200 import distributed, workload  # noqa: E402
from paper_2512_14946_b200.kvtier import Engine  # noqa: E402


def instance(name):
    """(arrays, tiers, space, params) of a large case, exactly as bench.py builds it."""
    if name == "c5":
        W = workload.build("c5")
        return W["arrays"], W["tiers"], W["space"], W["params"]
    world = {"ws8": 8, "ws2": 2}[name]
    Ws = [workload.build("c2", seed=7 + r) for r in range(world)]
    arrays = distributed.merge_rank_profiles([w["arrays"] for w in Ws])
    tiers = workload.three_tiers(int(arrays.orig.sum()), Ws[0]["cfg"]["gpu_frac"], 0.30)
    return arrays, tiers, Ws[0]["space"], Ws[0]["params"]


def input_hash(arrays):
    h = hashlib.sha256()
    for a in (arrays.orig, arrays.freq, arrays.goff, arrays.grid, arrays.qual, arrays.has):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update("\n".join(arrays.ids).encode())
    return h.hexdigest()


def main():
    cases = sys.argv[1:] or ["ws2", "c5", "ws8"]
    ref = Engine(A.Abi(os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so"), "ref_", codec=False))
    for name in cases:
        arrays, tiers, space, params = instance(name)
        ps = ref.pset(arrays)
        st = ref.store(tiers, arrays.n, space)
        t0 = time.perf_counter()
        acts = st.insert_joint(ps, space, params, np.arange(arrays.n, dtype=np.int32))
        dt = time.perf_counter() - t0
        snap = st.snapshot()
        pre = ""
        out = {}
        out[pre + "input_sha256"] = np.array(input_hash(arrays))
        out[pre + "actions"] = acts
        out[pre + "snapshot"] = snap
        out[pre + "occupancy"] = st.occupancy()
        out[pre + "utility"] = np.float64(st.placement_utility(ps, space, params))
        out[pre + "residents"] = np.concatenate([np.asarray(r, np.int32) for r in st.residents()])
        out[pre + "resident_counts"] = np.array([len(r) for r in st.residents()], np.int64)
        out[pre + "ref_seconds"] = np.float64(dt)
        print(f"{name}: {arrays.n} contexts, {len(acts)} actions, reference insert_joint {dt:.1f} s", flush=True)
        np.savez_compressed(os.path.join(HERE, f"large_placement_{name}.npz"), **out)


if __name__ == "__main__":
    main()
