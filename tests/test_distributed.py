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


def _worker_records(rank, world, port, out_dir):
    """bench.py's per-step rank logic (distributed.RankPlacement): record
    all-gathered over the process group, merged by the engine (the CPU
    restatement orc_pset_merge here, kvt_pset_merge on the GPU), replicated
    greedy over every context. Two steps, the second refilling the merged
    set in place."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from paper_2512_14946_b200 import _abi as A
    from paper_2512_14946_b200.kvtier import Engine
    from conftest import ORACLE_LIB
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W = workload.build("c3", n_ctx=N_LOCAL, seed=7 + rank)
    eng = Engine(A.Abi(ORACLE_LIB, "orc_", codec=False))
    rp = distributed.RankPlacement(eng, W["arrays"])
    out = {}
    for step in range(2):
        rp.upload()
        ps = rp.exchange()
        # tier budgets from the merged set's total bytes (every rank holds it)
        sc = eng.score_candidates(ps, workload.three_tiers(1, 0.1, 0.3), W["space"], W["params"])
        total = int(sc["size"][:, 0].sum())  # ratio index 0 = 1.0: the original sizes
        tiers = workload.three_tiers(total, W["cfg"]["gpu_frac"], 0.30)
        st = eng.store(tiers, ps.arrays.n, W["space"])
        acts = st.insert_joint(ps, W["space"], W["params"], np.arange(ps.arrays.n))
        out[f"acts{step}"] = acts
        out[f"snap{step}"] = st.snapshot()
        out[f"size{step}"] = sc["size"]
    np.savez(os.path.join(out_dir, f"rec{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_record_exchange_rank_logic(tmp_path, world):
    mp.start_processes(_worker_records, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    r = [np.load(tmp_path / f"rec{i}.npz") for i in range(world)]
    Ws = [workload.build("c3", n_ctx=N_LOCAL, seed=7 + i) for i in range(world)]
    cat = distributed.merge_rank_profiles([w["arrays"] for w in Ws])
    acts, snap = _run_greedy(cat, Ws[0])
    assert len(acts) > cat.n
    for i in range(world):
        for step in range(2):
            assert np.array_equal(r[i][f"acts{step}"], acts), (i, step)
            assert np.array_equal(r[i][f"snap{step}"], snap), (i, step)


def test_record_roundtrip_single_process():
    """pack_record + orc_pset_merge(world=1 and a hand-stacked world=3) ==
    pset_create on the same rows (every candidate table identical)."""
    from paper_2512_14946_b200 import _abi as A
    from paper_2512_14946_b200.kvtier import Engine, MergedPSet
    from conftest import ORACLE_LIB
    eng = Engine(A.Abi(ORACLE_LIB, "orc_", codec=False))
    Ws = [workload.build("c3", n_ctx=N_LOCAL, seed=7 + i) for i in range(3)]
    recs = [distributed.pack_record(eng.abi, w["arrays"]) for w in Ws]
    assert len({len(x) for x in recs}) == 1 and len(recs[0]) % 256 == 0
    M, g = Ws[0]["arrays"].M, int(Ws[0]["arrays"].goff[-1])
    for world in (1, 3):
        buf = np.concatenate(recs[:world])
        ps = MergedPSet(eng, world * N_LOCAL).merge(buf, world, N_LOCAL, g, M)
        ref = eng.pset(distributed.merge_rank_profiles([w["arrays"] for w in Ws[:world]]) if world > 1
                       else Ws[0]["arrays"])
        tiers = workload.three_tiers(10 ** 12, 0.1, 0.3)
        a = eng.score_candidates(ps, tiers, Ws[0]["space"], Ws[0]["params"])
        b = eng.score_candidates(ref, tiers, Ws[0]["space"], Ws[0]["params"])
        for k in a:
            assert np.array_equal(a[k], b[k]), (world, k)


@pytest.mark.parametrize("n,world", [(10, 3), (1000, 8), (7, 1)])
def test_shard_partitions(n, world):
    got = [distributed.shard(n, world, r) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
