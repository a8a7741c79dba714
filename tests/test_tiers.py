"""Tier-move executor: batched moves between the GPU tier
(device blobs) and the CPU tier (pinned host arena). CPU test: the oracle's
memcpy restatement of the batch semantics; GPU tests: device->host->device
round trips of real compressed blobs are bit-exact, moves are ordered after
the compress that produced the blob (same handle stream, no explicit sync),
and pieces > 8 MiB / many small moves / zero-byte moves work."""
import ctypes as C

import numpy as np
import pytest

from paper_2512_14946_b200 import _abi as A


def test_oracle_moves_copy_every_batch_entry(oracle_abi):
    rng = np.random.default_rng(0)
    srcs = [rng.integers(0, 255, n, dtype=np.uint8) for n in (1, 17, 4096, 0, 100000)]
    dsts = [np.zeros(len(s_), np.uint8) for s_ in srcs]
    moves = (A.Move * len(srcs))(*[A.Move(A.ptr(s_), A.ptr(d), len(s_), A.KVT_MOVE_H2H, 0) for s_, d in zip(srcs, dsts)])
    assert oracle_abi.tier_moves(None, moves, len(srcs)) == A.KVT_OK
    assert all(np.array_equal(s_, d) for s_, d in zip(srcs, dsts))
    bad = (A.Move * 1)(A.Move(None, A.ptr(dsts[0]), 5, A.KVT_MOVE_H2H, 0))
    assert oracle_abi.tier_moves(None, bad, 1) != A.KVT_OK


@pytest.mark.gpu
def test_gpu_blob_round_trip_through_host_tier(gpu_abi):
    import torch

    from paper_2512_14946_b200.kvtier import Engine
    from paper_2512_14946_b200.tiers import HostArena, TierExecutor, host_moves_bytes
    eng = Engine(gpu_abi)
    s = A.KvShape(4, 8, 2048, 128)
    n = s.L * s.H * s.T * s.D
    k = torch.empty(n, dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    eng.abi.check(eng.abi.kv_generate(eng.h, C.byref(s), 3, 1, A.ptr(k), A.ptr(v)))
    blobs = []
    for meth, ratio in (("knorm-q4", 0.2), ("keydiff", 0.5), ("snapkv-q8", 0.4)):
        cfg = A.CodecCfg()
        eng.abi.check(eng.abi.codec_plan(meth.encode(), ratio, C.byref(s), C.byref(cfg)))
        m = A.BlobMap()
        eng.abi.check(eng.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
        ws = torch.empty(eng.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg)), dtype=torch.uint8, device="cuda")
        b = torch.zeros(m.total_bytes, dtype=torch.uint8, device="cuda")
        eng.abi.check(eng.abi.compress(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws), A.ptr(b)))
        blobs.append((b, ws))
    arena = HostArena(eng.abi, sum(b.numel() for b, _ in blobs) + 4096)
    ex = TierExecutor(eng, arena)
    placed = [(i, 1 + (i % 2), b.data_ptr(), b.numel()) for i, (b, _) in enumerate(blobs)] + [(9, 0, 0, 123)]
    moves = ex.moves_for(placed)  # the GPU-tier context (tier 0) does not move
    assert len(moves) == 3 and host_moves_bytes(moves) == sum(b.numel() for b, _ in blobs)
    ex.run(moves)  # no sync: ordered after the compresses on the handle stream
    eng.abi.check(eng.abi.sync(eng.h))
    for (b, _), mv in zip(blobs, moves):
        host = np.ctypeslib.as_array((C.c_uint8 * mv.bytes).from_address(mv.dst))
        assert np.array_equal(host, b.cpu().numpy())
    back = [torch.zeros_like(b) for b, _ in blobs]
    up = [A.Move(mv.dst, t.data_ptr(), mv.bytes, A.KVT_MOVE_H2D, 0) for mv, t in zip(moves, back)]
    ex.run(up)
    eng.abi.check(eng.abi.sync(eng.h))
    for (b, _), t in zip(blobs, back):
        assert torch.equal(b, t)
    arena.close()


def test_ssd_tier_file_round_trip(tmp_path):
    """kvt_tier_file_* (host code, no GPU needed): aligned pieces take
    O_DIRECT where the file system allows it, unaligned ones the buffered
    descriptor; every byte reads back."""
    import paper_2512_14946_b200 as pkg
    from paper_2512_14946_b200.tiers import SsdTier
    abi = pkg.product()
    rng = np.random.default_rng(1)
    sizes = [4096 * 300, 70 << 20, 12345, 0, 4096]
    bufs = []
    for n in sizes:  # 4 KiB-aligned host buffers
        raw = np.zeros(n + 8192, np.uint8)
        off = (-raw.ctypes.data) % 4096
        b = raw[off:off + n]
        b[:] = rng.integers(0, 255, n, dtype=np.uint8)
        bufs.append((raw, b))
    ssd = SsdTier(abi, str(tmp_path / "ssd.tier"), sum(sizes) + 10 * 4096, threads=4)
    offs = [ssd.alloc(n) for n in sizes]
    ssd.write([(b.ctypes.data, n, o) for (_, b), n, o in zip(bufs, sizes, offs)])
    back = [np.zeros(n + 8192, np.uint8) for n in sizes]
    views = [r[(-r.ctypes.data) % 4096:][:n] for r, n in zip(back, sizes)]
    ssd.read([(v.ctypes.data, n, o) for v, n, o in zip(views, sizes, offs)])
    for (_, b), v in zip(bufs, views):
        assert np.array_equal(b, v)
    ssd.close()
    assert not (tmp_path / "ssd.tier").exists()


def test_net_placement_folds_actions_into_the_snapshot(oracle_abi):
    """The executor's view of a batch (its action list folded in order)
    equals the store's final state (proj/src/placement.cpp:213-221)."""
    from cases import random_instance
    from paper_2512_14946_b200.kvtier import Engine, sorted_tiers
    from paper_2512_14946_b200.tiers import net_placement
    eng = Engine(oracle_abi)
    arrays, tiers, space, params = random_instance(77, n_ctx=120, n_methods=3, n_tiers=3)
    ps = eng.pset(arrays)
    st = eng.store(tiers, arrays.n, space)
    acts = st.insert_joint(ps, space, params, np.arange(arrays.n))
    net = net_placement(acts, arrays.n, [t.tier_id for t in sorted_tiers(tiers)])
    snap = st.snapshot()
    assert np.array_equal(net["tier_index"], snap["tier_index"])
    assert np.array_equal(net["method"], snap["method"]) and np.array_equal(net["ratio"], snap["ratio"])
    assert net["inserts"].sum() == arrays.n and net["evicts"].sum() + net["recompress"].sum() == len(acts) - arrays.n
