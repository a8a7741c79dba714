"""pipeline.Codec on several CUDA streams: compress_split (scoring on one
stream, top-k + pack on another, handed over through a ring of score
buffers and CUDA events) must write the same blob bytes as kvt_compress on
one stream, including when more contexts than ring slots are in flight;
and the stream planner is pure host logic (CPU)."""
import ctypes as C

import pytest
import torch

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import Engine
from paper_2512_14946_b200.pipeline import Codec, split_plan

CASES = [("snapkv-q4", 0.2), ("snapkv", 0.3), ("snapkv-q8", 1.0), ("knorm-q8", 0.5), ("keydiff-q4", 0.15),
         ("snapkv-q2", 0.1)]


@pytest.mark.gpu
def test_compress_split_matches_compress(gpu_abi):
    L, H, T = 2, 4, 1536
    streams = [torch.cuda.Stream() for _ in range(3)]
    lanes = [Engine(gpu_abi, stream=s.cuda_stream) for s in streams]
    ref_eng = Engine(gpu_abi)
    codec = Codec(lanes, L, H)
    codec.reserve(T, n_out=1)
    codec.attach_streams(streams, ring=2)
    s = A.KvShape(L, H, T, 128)
    n = L * H * T * 128
    kvs = []
    for ctx in range(len(CASES) * 2):
        k = torch.empty(n, dtype=torch.int16, device="cuda")
        v = torch.empty_like(k)
        ref_eng.abi.check(ref_eng.abi.kv_generate(ref_eng.h, C.byref(s), 7, ctx, A.ptr(k), A.ptr(v)))
        kvs.append((k, v))
    ref_eng.abi.check(ref_eng.abi.sync(ref_eng.h))
    torch.cuda.synchronize()
    # reference blobs: kvt_compress on the default engine, one at a time
    want = []
    for ctx, (k, v) in enumerate(kvs):
        method, ratio = CASES[ctx % len(CASES)]
        cfg, m, wsb = codec.plan(method, ratio, T)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        blob = torch.empty(m.total_bytes, dtype=torch.uint8, device="cuda")
        ref_eng.abi.check(ref_eng.abi.compress(ref_eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws),
                                               A.ptr(blob)))
        ref_eng.abi.check(ref_eng.abi.sync(ref_eng.h))
        want.append(blob.cpu())
    # split: all contexts queued before any host sync (ring of 2 < contexts in flight);
    # each blob copied out on its pack lane before the lane's output slot is reused
    got = [None] * len(kvs)
    for ctx, (k, v) in enumerate(kvs):
        method, ratio = CASES[ctx % len(CASES)]
        pl = 1 + ctx % 2
        nb = codec.compress_split(method, ratio, k, v, T, ctx, 0, pl)
        with torch.cuda.stream(streams[pl]):
            got[ctx] = codec._out[pl][0][:nb].clone()
    torch.cuda.synchronize()
    for ctx in range(len(kvs)):  # the blob's sections (gaps between them are never written)
        method, ratio = CASES[ctx % len(CASES)]
        cfg, m, _ = codec.plan(method, ratio, T)
        g, w = _sections(got[ctx], m, cfg.bits), _sections(want[ctx], m, cfg.bits)
        for name in w:
            assert torch.equal(g[name], w[name]), (method, ratio, name)


def _sections(b, m, bits):
    b = b.cpu()
    out = {"idx": b[m.idx_off:m.idx_off + m.idx_bytes], "kcode": b[m.kcode_off:m.kcode_off + m.kcode_bytes],
           "vcode": b[m.vcode_off:m.vcode_off + m.vcode_bytes]}
    if bits < 16:
        for n, o, sz in (("kscale", m.kscale_off, m.kparam_bytes), ("kzero", m.kzero_off, m.kparam_bytes),
                         ("vscale", m.vscale_off, m.vparam_bytes), ("vzero", m.vzero_off, m.vparam_bytes)):
            out[n] = b[o:o + sz]
    return out


def test_split_plan_puts_snapkv_scoring_on_lane0():
    ms = ["snapkv-q4", "knorm", "snapkv", "keydiff-q8", "snapkv-q4", "knorm-q4"]
    rs = [0.2, 0.4, 1.0, 0.3, 0.5, 0.1]
    plan = split_plan(ms, rs, [8192] * len(ms), 3, snap_sms=64)
    for (sl, pl), m, r in zip(plan, ms, rs):
        assert pl in (1, 2)
        assert sl == (0 if m.startswith("snapkv") and r < 1.0 else None)
    assert {pl for _, pl in plan} == {1, 2}  # balanced over both pack lanes
