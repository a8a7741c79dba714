"""The N > 1 path on CPU (gloo, world_size 2, 127.0.0.1): the profile
all-gather, the context shards and the replicated greedy. Every rank must
end with the same global profile set and the same action list, equal to a
single-process run over the concatenated profiles, and the shards must
partition the contexts. The greedy runs on the CPU oracle engine here (the
CUDA engine is the same ABI; its parity with the oracle is
tests/test_gpu_placement.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_14946_b200 import distributed, workload
from paper_2512_14946_b200.kvtier import ProfileArrays

N_LOCAL = 40


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_greedy(arrays, W):
    from paper_2512_14946_b200 import _abi as A
    from paper_2512_14946_b200.kvtier import Engine
    from conftest import ORACLE_LIB
    eng = Engine(A.Abi(ORACLE_LIB, "orc_", codec=False))
    tiers = workload.three_tiers(int(arrays.orig.sum()), W["cfg"]["gpu_frac"], 0.30)
    ps = eng.pset(arrays)
    st = eng.store(tiers, arrays.n, W["space"])
    acts = st.insert_joint(ps, W["space"], W["params"], np.arange(arrays.n))
    return acts, st.snapshot()


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W = workload.build("c3", n_ctx=N_LOCAL, seed=7 + rank)
    arrays = distributed.gather_profiles(W["arrays"])
    acts, snap = _run_greedy(arrays, W)
    lo, hi = distributed.shard(arrays.n, world, rank)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), orig=arrays.orig, qual=arrays.qual, freq=arrays.freq,
             acts=acts, snap=snap, lo=lo, hi=hi, ids=np.array(arrays.ids))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_shard_and_replicated_greedy(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(world)]
    # every rank holds the same global profile set and computed the same placement
    for k in ("orig", "qual", "freq", "acts", "snap", "ids"):
        assert np.array_equal(r[0][k], r[1][k]), k
    # = a single process over the concatenated per-rank profiles
    Ws = [workload.build("c3", n_ctx=N_LOCAL, seed=7 + i) for i in range(world)]
    G = len(Ws[0]["arrays"].grid) // N_LOCAL
    cat = ProfileArrays.uniform_grid(
        distributed.context_ids(N_LOCAL, world), np.concatenate([w["arrays"].orig for w in Ws]),
        np.concatenate([w["arrays"].freq for w in Ws]), Ws[0]["arrays"].grid[:G],
        np.concatenate([w["arrays"].qual.reshape(N_LOCAL, -1, G) for w in Ws]),
        np.concatenate([w["arrays"].has for w in Ws]))
    acts, snap = _run_greedy(cat, Ws[0])
    assert np.array_equal(acts, r[0]["acts"]) and np.array_equal(snap, r[0]["snap"])
    assert len(acts) > cat.n  # the budgets force overflow steps, not just inserts
    # shards partition the contexts, rank-major like the merged id order
    ranges = sorted((int(x["lo"]), int(x["hi"])) for x in r)
    assert ranges[0][0] == 0 and ranges[-1][1] == world * N_LOCAL and ranges[0][1] == ranges[1][0]
    assert list(r[0]["ids"]) == sorted(r[0]["ids"], key=lambda s: s.encode())


@pytest.mark.parametrize("n,world", [(10, 3), (1000, 8), (7, 1)])
def test_shard_partitions(n, world):
    got = [distributed.shard(n, world, r) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
