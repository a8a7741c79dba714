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
