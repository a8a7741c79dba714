"""CUDA codec vs the codec oracle (oracle/orc_codec.c), all bit-exact:
synthetic KV, knorm/keydiff/snapkv scores, top-k indices, packed codes +
fp16 params, dequantised KV."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import Engine

pytestmark = pytest.mark.gpu



@pytest.fixture(scope="module")
def gpu(gpu_abi):
    return Engine(gpu_abi)


@pytest.fixture(scope="module")
def orc(oracle_abi):
    return Engine(oracle_abi)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t, dtype):
    return t.cpu().numpy().view(dtype)


def plan(abi, method, ratio, s):
    cfg = A.CodecCfg()
    abi.check(abi.codec_plan(method.encode(), ratio, C.byref(s), C.byref(cfg)))
    return cfg


def gen(eng, s, seed=9, ctx=3, on_gpu=True):
    n = s.L * s.H * s.T * s.D
    if on_gpu:
        k = torch.empty(n, dtype=torch.int16, device="cuda")
        v = torch.empty_like(k)
        eng.abi.check(eng.abi.kv_generate(eng.h, C.byref(s), seed, ctx, A.ptr(k), A.ptr(v)))
        eng.abi.check(eng.abi.sync(eng.h))
        return k, v
    k = np.zeros(n, np.uint16)
    v = np.zeros(n, np.uint16)
    eng.abi.check(eng.abi.kv_generate(None, C.byref(s), seed, ctx, A.ptr(k), A.ptr(v)))
    return k, v


SHAPES = [A.KvShape(2, 2, 300, 128), A.KvShape(1, 3, 1000, 128), A.KvShape(3, 1, 129, 128)]
# compress also at Llama chunk length (T = 8192: 1024 tokens per cluster CTA),
# a ragged length and a length below the cluster size
PACK_SHAPES = SHAPES + [A.KvShape(1, 2, 8192, 128), A.KvShape(2, 1, 4097, 128), A.KvShape(1, 1, 5, 128)]


@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_kv_generate_bitexact(gpu, orc, si):
    s = SHAPES[si]
    kg, vg = gen(gpu, s)
    ko, vo = gen(orc, s, on_gpu=False)
    assert np.array_equal(host(kg, np.uint16), ko) and np.array_equal(host(vg, np.uint16), vo)


def scores(eng, s, cfg, k, on_gpu):
    if on_gpu:
        out = torch.empty(s.L * s.H * s.T, dtype=torch.float32, device="cuda")
        eng.abi.check(eng.abi.token_scores(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(out)))
        eng.abi.check(eng.abi.sync(eng.h))
        return out.cpu().numpy()
    out = np.zeros(s.L * s.H * s.T, np.float32)
    eng.abi.check(eng.abi.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(out)))
    return out


@pytest.mark.parametrize("si", range(len(SHAPES)))
@pytest.mark.parametrize("method", ["knorm", "keydiff"])
def test_scores_bitexact(gpu, orc, si, method):
    s = SHAPES[si]
    kg, _ = gen(gpu, s)
    ko, _ = gen(orc, s, on_gpu=False)
    cfg = plan(orc.abi, method, 0.3, s)
    sg, so = scores(gpu, s, cfg, kg, True), scores(orc, s, cfg, ko, False)
    assert np.array_equal(sg.view(np.uint32), so.view(np.uint32))


# keydiff prefix lengths: 1 token, 49 rows per cluster CTA, Llama chunk,
# ragged lengths, 2,048 rows per CTA
KD_SHAPES = [A.KvShape(1, 2, 1, 128), A.KvShape(2, 3, 385, 128), A.KvShape(1, 3, 8192, 128),
             A.KvShape(2, 1, 9216, 128), A.KvShape(1, 2, 9217, 128), A.KvShape(3, 2, 4097, 128),
             A.KvShape(1, 1, 16384, 128), A.KvShape(1, 1, 6657, 128)]


@pytest.mark.parametrize("si", range(len(KD_SHAPES)))
def test_keydiff_lengths_bitexact(gpu, orc, si):
    s = KD_SHAPES[si]
    kg, _ = gen(gpu, s)
    ko, _ = gen(orc, s, on_gpu=False)
    cfg = plan(orc.abi, "keydiff", 0.3, s)
    sg, so = scores(gpu, s, cfg, kg, True), scores(orc, s, cfg, ko, False)
    assert np.array_equal(sg.view(np.uint32), so.view(np.uint32))


def topk(eng, s, cfg, sc, on_gpu):
    if on_gpu:
        out = torch.empty(s.L * s.H * cfg.keep, dtype=torch.int32, device="cuda")
        eng.abi.check(eng.abi.topk(eng.h, C.byref(s), C.byref(cfg), A.ptr(sc), A.ptr(out)))
        eng.abi.check(eng.abi.sync(eng.h))
        return out.cpu().numpy()
    out = np.zeros(s.L * s.H * cfg.keep, np.int32)
    eng.abi.check(eng.abi.topk(None, C.byref(s), C.byref(cfg), A.ptr(sc), A.ptr(out)))
    return out


# snapkv prefix lengths (8 tiles = 1,024 tokens per cluster CTA in the
# smem-E configuration): one tile, 1 token, several tiles in one CTA, an
# 8-CTA cluster (T = 8192), ragged last tiles and blocks, a 9-CTA cluster
# (8225), 16 CTAs (16384: the longest smem-E prefix is 16,384 tokens), the
# global-E configuration (T = 20000: 10 CTAs x 16 tiles, E in per-SM L2
# slots, votes on the CUDA cores), and prefixes of length 0 (all window)
SNAP_SHAPES = SHAPES + [A.KvShape(1, 1, 33, 128), A.KvShape(1, 2, 8192, 128), A.KvShape(2, 1, 4097, 128),
                        A.KvShape(1, 1, 8224, 128), A.KvShape(1, 1, 8225, 128), A.KvShape(1, 2, 16384, 128),
                        A.KvShape(1, 2, 32, 128), A.KvShape(1, 1, 20, 128), A.KvShape(1, 2, 20000, 128)]


@pytest.mark.parametrize("si", range(len(SNAP_SHAPES)))
def test_snapkv_scores_bitexact(gpu, orc, si):
    """int8 tensor-core logits + fixed-point softmax votes == the oracle, bit for bit."""
    s = SNAP_SHAPES[si]
    kg, _ = gen(gpu, s)
    ko, _ = gen(orc, s, on_gpu=False)
    cfg = plan(orc.abi, "snapkv", 0.3, s)
    sg, so = scores(gpu, s, cfg, kg, True), scores(orc, s, cfg, ko, False)
    assert np.array_equal(sg.view(np.uint32), so.view(np.uint32))


def window_queries(s, cfg, seed, spread=1.0):
    """Caller-supplied observation-window queries, bf16 [L][H*G][W][128]:
    random normal rows with a few large channels (real queries are peaky)."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((s.L, s.H * cfg.q_heads, cfg.window, 128)).astype(np.float32) * np.float32(spread)
    q[..., 3] *= np.float32(8.0)
    q[..., 77] *= np.float32(-5.0)
    return (q.view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("si", [0, 1, 4, 5, 7, 9, 11])
@pytest.mark.parametrize("spread", [1.0, 30.0])
def test_snapkv_caller_queries_bitexact(gpu, orc, si, spread):
    """snapkv over the caller's observation-window queries
    instead of the synthetic ones: token_scores and compress equal the oracle."""
    s = SNAP_SHAPES[si]
    kg, vg = gen(gpu, s)
    ko, vo = gen(orc, s, on_gpu=False)
    cfg = plan(orc.abi, "snapkv-q4", 0.2, s)
    q = window_queries(s, cfg, si, spread)
    qg = dev(q.view(np.int16))
    out = torch.empty(s.L * s.H * s.T, dtype=torch.float32, device="cuda")
    gpu.abi.check(gpu.abi.token_scores(gpu.h, C.byref(s), C.byref(cfg), A.ptr(kg), A.ptr(qg), A.ptr(out)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    want = np.zeros(s.L * s.H * s.T, np.float32)
    orc.abi.check(orc.abi.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(ko), A.ptr(q), A.ptr(want)))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    synth = scores(orc, s, cfg, ko, False)
    if s.T > cfg.window + 1:
        assert not np.array_equal(synth, want)  # the queries matter
    # compress with the caller's queries: same blob as the oracle's
    m = A.BlobMap()
    orc.abi.check(orc.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    ws = torch.empty(gpu.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg)), dtype=torch.uint8, device="cuda")
    bg = torch.zeros(m.total_bytes, dtype=torch.uint8, device="cuda")
    gpu.abi.check(gpu.abi.compress(gpu.h, C.byref(s), C.byref(cfg), A.ptr(kg), A.ptr(vg), A.ptr(qg), A.ptr(ws),
                                   A.ptr(bg)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    wso = np.zeros(orc.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg)), np.uint8)
    bo = np.zeros(m.total_bytes, np.uint8)
    orc.abi.check(orc.abi.compress(None, C.byref(s), C.byref(cfg), A.ptr(ko), A.ptr(vo), A.ptr(q), A.ptr(wso),
                                   A.ptr(bo)))
    assert np.array_equal(bg.cpu().numpy(), bo)


@pytest.mark.parametrize("T", [32 + 300, 32 + 129, 32 + 8192])
@pytest.mark.parametrize("spread", [3.0, 30.0])
def test_snapkv_k_groups_bitexact(gpu, orc, T, spread):
    """spec v4 per-16-token K scales on structured keys (an all-zero group, a
    huge outlier row whose logit factor hits the 1/4 cap, tiny and constant
    groups, -0, ragged last group and block) with caller queries: scores
    equal the oracle bit for bit, through the clamped and clamp-free E paths."""
    from test_codec_oracle import _snap_groups_k, _snap_queries
    s = A.KvShape(1, 2, T, 128)
    k = _snap_groups_k(1, 2, T)
    cfg = plan(orc.abi, "snapkv", 0.5, s)
    q = _snap_queries(s, cfg, spread=spread)
    want = np.zeros(2 * T, np.float32)
    orc.abi.check(orc.abi.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(q), A.ptr(want)))
    kg, qg = dev(k.reshape(-1).view(np.int16)), dev(q.reshape(-1).view(np.int16))
    out = torch.empty(2 * T, dtype=torch.float32, device="cuda")
    gpu.abi.check(gpu.abi.token_scores(gpu.h, C.byref(s), C.byref(cfg), A.ptr(kg), A.ptr(qg), A.ptr(out)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("method", ["knorm", "keydiff"])
def test_scores_denormal_keys_bitexact(gpu, orc, method):
    """bf16 subnormal, zero and -0 keys (rows of them, and rows mixing them
    with normal channels): scores equal the oracle's bit for bit (no flush
    to zero anywhere on the path)."""
    s = A.KvShape(1, 2, 300, 128)
    k, _ = gen(orc, s, on_gpu=False)
    x = k.reshape(2, 300, 128).copy()
    rng = np.random.default_rng(3)
    sub = rng.integers(1, 0x80, size=(2, 100, 128)).astype(np.uint16)  # bf16 subnormals: exponent 0
    sub |= (rng.integers(0, 2, size=sub.shape).astype(np.uint16) << 15)
    x[:, 50:150] = sub
    x[:, 160:170] = 0x8000  # -0 rows
    x[:, 170:180, :64] = sub[:, :10, :64]
    x = x.reshape(-1)
    cfg = plan(orc.abi, method, 0.3, s)
    want = np.zeros(2 * 300, np.float32)
    orc.abi.check(orc.abi.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(x), None, A.ptr(want)))
    kg = dev(x.view(np.int16))
    out = torch.empty(2 * 300, dtype=torch.float32, device="cuda")
    gpu.abi.check(gpu.abi.token_scores(gpu.h, C.byref(s), C.byref(cfg), A.ptr(kg), None, A.ptr(out)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_knorm_keep_low_flag(gpu, orc, si):
    """KVT_CODEC_KNORM_KEEP_LOW (the cited knorm paper keeps low-norm keys;
    PAPER.md:637 drops them): scores are the negated norms, bit-exact."""
    s = SHAPES[si]
    kg, _ = gen(gpu, s)
    ko, _ = gen(orc, s, on_gpu=False)
    cfg = plan(orc.abi, "knorm", 0.3, s)
    hi = scores(gpu, s, cfg, kg, True)
    cfg.flags = A.KVT_CODEC_KNORM_KEEP_LOW
    lo_g, lo_o = scores(gpu, s, cfg, kg, True), scores(orc, s, cfg, ko, False)
    assert np.array_equal(lo_g.view(np.uint32), lo_o.view(np.uint32))
    assert np.array_equal(lo_g, -hi)


@pytest.mark.parametrize("sms", ["1", "16", "64", "100"])
def test_snapkv_sm_budget_same_scores(gpu, sms, monkeypatch):
    """KVT_SNAP_SMS (the bench's SM budget for snapkv's persistent clusters)
    changes only how many clusters loop over the slices: scores identical."""
    s = A.KvShape(2, 4, 3000, 128)  # 6-CTA clusters, 8 slices
    kg, _ = gen(gpu, s)
    cfg = plan(gpu.abi, "snapkv", 0.3, s)
    want = scores(gpu, s, cfg, kg, True)
    monkeypatch.setenv("KVT_SNAP_SMS", sms)
    assert np.array_equal(scores(gpu, s, cfg, kg, True).view(np.uint32), want.view(np.uint32))


def test_snapkv_rejects_too_long_prefix(gpu):
    s = A.KvShape(1, 1, 32768 + 32 + 1, 128)  # prefix of 32769 tokens
    cfg = plan(gpu.abi, "snapkv", 0.3, s)
    k = torch.zeros(s.L * s.H * s.T * s.D, dtype=torch.int16, device="cuda")
    out = torch.empty(s.L * s.H * s.T, dtype=torch.float32, device="cuda")
    with pytest.raises(A.AbiError):
        gpu.abi.check(gpu.abi.token_scores(gpu.h, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(out)))


@pytest.mark.parametrize("keep_ratio", [0.001, 0.2, 0.5, 1.0])
def test_topk_bitexact_with_ties(gpu, orc, keep_ratio):
    s = A.KvShape(2, 3, 5000, 128)
    rng = np.random.default_rng(4)
    sc = rng.integers(0, 50, s.L * s.H * s.T).astype(np.float32)  # heavy ties
    sc[::7] = -0.0
    sc[1::11] = np.float32(-3.5)
    sc[5000:10000] = rng.standard_normal(5000).astype(np.float32)
    cfg = plan(orc.abi, "knorm", keep_ratio, s)
    assert np.array_equal(topk(gpu, s, cfg, dev(sc), True), topk(orc, s, cfg, sc, False))


# top-k key distributions for the adaptive first radix digit: every key
# equal, keys differing only in the last mantissa bits, +inf window scores
# mixed in, the full signed range, a slice too long for smem keys, and an
# odd-length slice whose keys + staged indices fit smem at small keep only
TOPK_CASES = ["equal", "ulps", "inf", "wide", "long", "odd"]


@pytest.mark.parametrize("case", TOPK_CASES)
@pytest.mark.parametrize("keep_ratio", [0.01, 0.37, 0.9])
def test_topk_key_distributions(gpu, orc, case, keep_ratio):
    T = {"long": 41000, "odd": 30001}.get(case, 3000)
    s = A.KvShape(1, 2, T, 128)
    rng = np.random.default_rng(7)
    n = s.L * s.H * s.T
    if case == "equal":
        sc = np.full(n, 1.25, np.float32)
    elif case == "ulps":
        sc = (np.float32(3.0).view(np.uint32) + rng.integers(0, 5, n).astype(np.uint32)).view(np.float32)
    elif case == "inf":
        sc = rng.standard_normal(n).astype(np.float32)
        sc[rng.random(n) < 0.05] = np.inf
    elif case == "odd":
        sc = rng.standard_normal(n).astype(np.float32)
    else:
        sc = (rng.standard_normal(n) * np.float32(1e30)).astype(np.float32)
        sc[::13] = -0.0
        sc[::17] = 0.0
    cfg = plan(orc.abi, "knorm", keep_ratio, s)
    assert np.array_equal(topk(gpu, s, cfg, dev(sc), True), topk(orc, s, cfg, sc, False))


def compress(eng, s, cfg, k, v, on_gpu):
    m = A.BlobMap()
    eng.abi.check(eng.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    wsb = eng.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg))
    if on_gpu:
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        blob = torch.zeros(m.total_bytes, dtype=torch.uint8, device="cuda")
        eng.abi.check(eng.abi.compress(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws), A.ptr(blob)))
        eng.abi.check(eng.abi.sync(eng.h))
    else:
        ws = np.zeros(wsb, np.uint8)
        blob = np.zeros(m.total_bytes, np.uint8)
        eng.abi.check(eng.abi.compress(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws), A.ptr(blob)))
    return blob, m


def blob_sections(b, m, bits):
    b = b.cpu().numpy() if isinstance(b, torch.Tensor) else b
    out = {"idx": b[m.idx_off:m.idx_off + m.idx_bytes], "kcode": b[m.kcode_off:m.kcode_off + m.kcode_bytes],
           "vcode": b[m.vcode_off:m.vcode_off + m.vcode_bytes]}
    if bits < 16:
        for n, o, sz in (("kscale", m.kscale_off, m.kparam_bytes), ("kzero", m.kzero_off, m.kparam_bytes),
                         ("vscale", m.vscale_off, m.vparam_bytes), ("vzero", m.vzero_off, m.vparam_bytes)):
            out[n] = b[o:o + sz]
    return out


@pytest.mark.parametrize("si", range(len(PACK_SHAPES)))
@pytest.mark.parametrize("method,ratio", [("knorm-q8", 0.3), ("keydiff-q4", 0.2), ("knorm-q2", 0.1),
                                          ("keydiff", 0.4), ("knorm-q4", 0.02), ("knorm-q8", 0.5),
                                          ("keydiff-q8", 1.0), ("knorm", 1.0), ("snapkv", 1.0),
                                          ("snapkv-q4", 0.2), ("snapkv-q8", 0.4)])
def test_compress_unpack_bitexact(gpu, orc, si, method, ratio):
    """compress = scores + top-k + pack, then unpack: blobs and dequantised
    KV equal the oracle's. Identity configurations (every token at 16 bits)
    have no blob: nothing is launched and unpack refuses (the source is the
    decompressed KV)."""
    s = PACK_SHAPES[si]
    kg, vg = gen(gpu, s)
    ko, vo = gen(orc, s, on_gpu=False)
    cfg = plan(orc.abi, method, ratio, s)
    l0 = gpu.abi.launch_count(gpu.h)
    bg, m = compress(gpu, s, cfg, kg, vg, True)
    bo, _ = compress(orc, s, cfg, ko, vo, False)
    if m.identity:
        assert cfg.keep == s.T and cfg.bits == 16 and m.total_bytes == 0
        assert gpu.abi.launch_count(gpu.h) == l0
        for e, b in ((gpu, bg), (orc, bo)):
            with pytest.raises(A.AbiError):
                e.abi.check(e.abi.unpack(e.h if e is gpu else None, C.byref(s), C.byref(cfg), A.ptr(b), None, None))
        return
    sg, so = blob_sections(bg, m, cfg.bits), blob_sections(bo, m, cfg.bits)
    for name in so:
        assert np.array_equal(sg[name], so[name]), name
    n = s.L * s.H * cfg.keep * 128
    kug = torch.empty(n, dtype=torch.int16, device="cuda")
    vug = torch.empty_like(kug)
    gpu.abi.check(gpu.abi.unpack(gpu.h, C.byref(s), C.byref(cfg), A.ptr(bg), A.ptr(kug), A.ptr(vug)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    kuo = np.zeros(n, np.uint16)
    vuo = np.zeros(n, np.uint16)
    orc.abi.check(orc.abi.unpack(None, C.byref(s), C.byref(cfg), A.ptr(bo), A.ptr(kuo), A.ptr(vuo)))
    assert np.array_equal(host(kug, np.uint16), kuo) and np.array_equal(host(vug, np.uint16), vuo)


@pytest.mark.parametrize("shape,group", [((2, 3, 300), 1), ((2, 3, 300), 4), ((1, 4, 8192), 3),
                                         ((3, 1, 129), 2), ((2, 2, 4097), 5)])
@pytest.mark.parametrize("method,ratio", [("knorm-q8", 0.3), ("keydiff-q4", 0.2), ("knorm", 0.4),
                                          ("keydiff-q2", 1.0), ("knorm-q4", 0.02), ("keydiff", 1.0)])
def test_compress_slices_bitexact(gpu, orc, shape, group, method, ratio):
    """kvt_compress_slices over slice groups (ragged last group) writes the
    blob the oracle's whole-chunk compress writes, byte for byte."""
    s = A.KvShape(*shape, 128)
    S = s.L * s.H
    kg, vg = gen(gpu, s)
    ko, vo = gen(orc, s, on_gpu=False)
    cfg = plan(orc.abi, method, ratio, s)
    m = A.BlobMap()
    gpu.abi.check(gpu.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    ws = torch.empty(gpu.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg)), dtype=torch.uint8, device="cuda")
    bg = torch.zeros(max(1, m.total_bytes), dtype=torch.uint8, device="cuda")
    l0 = gpu.abi.launch_count(gpu.h)
    for s0 in range(0, S, group):
        gpu.abi.check(gpu.abi.compress_slices(gpu.h, C.byref(s), C.byref(cfg), A.ptr(kg), A.ptr(vg), s0,
                                              min(group, S - s0), A.ptr(ws), A.ptr(bg)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    if m.identity:
        assert gpu.abi.launch_count(gpu.h) == l0
        return
    bo, _ = compress(orc, s, cfg, ko, vo, False)
    sg, so = blob_sections(bg, m, cfg.bits), blob_sections(bo, m, cfg.bits)
    for name in so:
        assert np.array_equal(sg[name], so[name]), name


def test_compress_slices_rejects(gpu):
    s = A.KvShape(2, 2, 300, 128)
    kg, vg = gen(gpu, s)
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    blob = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    for method, s0, ns in (("snapkv-q4", 0, 2), ("knorm-q4", 3, 2), ("knorm-q4", -1, 1), ("knorm-q4", 0, -1)):
        cfg = plan(gpu.abi, method, 0.2, s)
        with pytest.raises(A.AbiError):
            gpu.abi.check(gpu.abi.compress_slices(gpu.h, C.byref(s), C.byref(cfg), A.ptr(kg), A.ptr(vg), s0, ns,
                                                  A.ptr(ws), A.ptr(blob)))


def test_full_llama_chunk_knorm_q4_properties(gpu, orc):
    """One full Llama-3.1-8B chunk (32 L x 8 H x 8192 T x 128, 1 GiB):
    knorm scores bit-exact to the oracle, top-k sorted and sized, and the
    unpacked KV within half a quantisation step of the kept originals."""
    s = A.KvShape(32, 8, 8192, 128)
    kg, vg = gen(gpu, s, seed=1, ctx=0)
    cfg = plan(orc.abi, "knorm-q4", 0.1, s)
    sg = scores(gpu, s, cfg, kg, True)
    ko, _ = gen(orc, A.KvShape(32, 8, 8192, 128), seed=1, ctx=0, on_gpu=False)
    so = scores(orc, s, cfg, ko, False)
    assert np.array_equal(sg.view(np.uint32), so.view(np.uint32))
    bg, m = compress(gpu, s, cfg, kg, vg, True)
    idx = bg[m.idx_off:m.idx_off + m.idx_bytes].view(torch.int32).reshape(256, cfg.keep)
    assert bool((idx[:, 1:] > idx[:, :-1]).all()) and int(idx.min()) >= 0 and int(idx.max()) < 8192
    n = 256 * cfg.keep * 128
    ku = torch.empty(n, dtype=torch.int16, device="cuda")
    vu = torch.empty_like(ku)
    gpu.abi.check(gpu.abi.unpack(gpu.h, C.byref(s), C.byref(cfg), A.ptr(bg), A.ptr(ku), A.ptr(vu)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    kk = kg.view(torch.bfloat16).float().reshape(256, 8192, 128)
    vv = vg.view(torch.bfloat16).float().reshape(256, 8192, 128)
    gi = idx.long()[..., None].expand(-1, -1, 128)
    kk = torch.gather(kk, 1, gi)
    vv = torch.gather(vv, 1, gi)
    kd = ku.view(torch.bfloat16).float().reshape(256, cfg.keep, 128)
    vd = vu.view(torch.bfloat16).float().reshape(256, cfg.keep, 128)
    vstep = (vv.amax(2, keepdim=True) - vv.amin(2, keepdim=True)) / 15
    assert bool(((vd - vv).abs() <= 0.51 * vstep * 1.002 + vv.abs() * 2 ** -7 + 1e-3).all())
    for g0 in range(0, cfg.keep, 128):
        seg = kk[:, g0:g0 + 128]
        kstep = (seg.amax(1, keepdim=True) - seg.amin(1, keepdim=True)) / 15
        assert bool(((kd[:, g0:g0 + 128] - seg).abs() <= 0.51 * kstep * 1.002 + seg.abs() * 2 ** -7 + 1e-3).all())


@pytest.mark.parametrize("bits", [2, 4, 8, 16])
def test_pack_extreme_values_bitexact(gpu, orc, bits):
    """Outlier KV (rows beyond fp16 range, tiny ranges far from zero, zeros,
    -0): groups whose parameters do not bound the codes take the exact FP64
    path; the blob still equals the oracle's byte for byte."""
    from test_codec_oracle import _extreme_kv
    s = A.KvShape(2, 2, 300, 128)
    k, v = _extreme_kv(2, 2, 300)
    cfg = plan(orc.abi, f"knorm-q{bits}" if bits < 16 else "knorm", 0.3 if bits < 16 else 0.5, s)
    cfg.bits = bits
    m = A.BlobMap()
    orc.abi.check(orc.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    rng = np.random.default_rng(bits)
    idx = np.sort(np.stack([np.stack([rng.choice(300, cfg.keep, replace=False) for _ in range(2)]) for _ in range(2)]),
                  axis=-1).astype(np.int32)
    bo = np.zeros(m.total_bytes, np.uint8)
    orc.abi.check(orc.abi.pack(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), A.ptr(idx), A.ptr(bo)))
    bg = torch.zeros(m.total_bytes, dtype=torch.uint8, device="cuda")
    kd, vd, idd = dev(k.view(np.int16)), dev(v.view(np.int16)), dev(idx)
    gpu.abi.check(gpu.abi.pack(gpu.h, C.byref(s), C.byref(cfg), A.ptr(kd), A.ptr(vd), A.ptr(idd), A.ptr(bg)))
    gpu.abi.check(gpu.abi.sync(gpu.h))
    sg, so = blob_sections(bg.cpu().numpy(), m, bits), blob_sections(bo, m, bits)
    for name in so:
        assert np.array_equal(sg[name], so[name]), name
