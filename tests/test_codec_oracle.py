"""Pins the codec oracle (oracle/orc_codec.c). The reference has no codec, so
parity is UNPINNED against the reference; the oracle is instead checked
against known answers derived from the spec and an independent numpy
restatement (tests/codec_ref.py)."""
import ctypes as C

import numpy as np
import pytest

from paper_2512_14946_b200 import _abi as A

import codec_ref as R


def shape(L, H, T, D=128):
    return A.KvShape(L, H, T, D)


def plan(abi, method, ratio, s):
    cfg = A.CodecCfg()
    abi.check(abi.codec_plan(method.encode(), ratio, C.byref(s), C.byref(cfg)))
    return cfg


@pytest.fixture(scope="module")
def lib(oracle_abi):
    L = oracle_abi.lib
    L.orc_f2h.restype = C.c_uint16
    L.orc_f2h.argtypes = [C.c_float]
    L.orc_h2f.restype = C.c_float
    L.orc_h2f.argtypes = [C.c_uint16]
    L.orc_f2bf.restype = C.c_uint16
    L.orc_f2bf.argtypes = [C.c_float]
    return oracle_abi


def test_half_and_bf16_rounding_match_numpy_torch(lib):
    import torch
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.standard_normal(3000).astype(np.float32) * np.float32(2.0) ** rng.integers(-30, 18, 3000).astype(np.float32),
        np.array([0.0, -0.0, 65504, 65519.99, 65520, 1e-8, 5.96e-8, 2.98e-8, 6.1e-5, -3.3e-6, 1 / 3], np.float32)])
    for v in vals:
        h = lib.lib.orc_f2h(float(v))
        assert h == np.float32(v).astype(np.float16).view(np.uint16), v
        assert lib.lib.orc_h2f(h) == np.float16(np.uint16(h).view(np.float16)).astype(np.float32) or np.isnan(v)
    t = torch.tensor(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    for v, want in zip(vals, t):
        assert lib.lib.orc_f2bf(float(v)) == want


def test_codec_plan_known_answers(lib):
    s = shape(32, 8, 8192)
    c = plan(lib, "knorm", 0.4, s)  # bf16 token drop, keep 0.4
    assert (c.scorer, c.bits, c.keep) == (A.KVT_SCORER_KNORM, 16, 3277)
    c = plan(lib, "keydiff-q4", 0.2, s)  # 4-bit: eff 0.265625 -> keep 0.7529
    assert (c.scorer, c.bits, c.keep) == (A.KVT_SCORER_KEYDIFF, 4, int(np.floor(0.2 / 0.265625 * 8192 + 0.5)))
    c = plan(lib, "keydiff-q4", 0.4, s)  # too big for 4 bits -> 8 bits
    assert c.bits == 8 and c.keep == int(np.floor(0.4 / (0.5 + 1 / 64) * 8192 + 0.5))
    c = plan(lib, "snapkv-q2", 0.9, s)  # -> bf16
    assert c.bits == 16 and c.keep == int(np.floor(0.9 * 8192 + 0.5))
    c = plan(lib, "snapkv", 0.0001, s)  # snapkv keeps at least its window
    assert c.keep == 32 and c.window == 32
    c = plan(lib, "knorm-q8", 1.0, s)
    assert c.bits == 16 and c.keep == 8192
    with pytest.raises(A.ValidationError):
        plan(lib, "h2o", 0.5, s)
    with pytest.raises(A.ValidationError):
        plan(lib, "knorm-q3", 0.5, s)


def test_blob_layout_sizes(lib):
    s = shape(2, 2, 300)
    for method, ratio in [("knorm-q4", 0.2), ("knorm-q8", 0.3), ("knorm-q2", 0.1), ("knorm", 0.5)]:
        c = plan(lib, method, ratio, s)
        m = A.BlobMap()
        lib.check(lib.blob_layout(C.byref(s), C.byref(c), C.byref(m)))
        S, k, b = 4, c.keep, c.bits
        assert m.idx_bytes == 4 * S * k
        if b == 16:
            assert m.kcode_bytes == m.vcode_bytes == 2 * S * k * 128
        else:
            ng = -(-k // 128)
            assert m.kcode_bytes == S * k * 128 * b // 8
            assert m.kparam_bytes == 2 * S * ng * 128 and m.vparam_bytes == 2 * S * k
        assert m.total_bytes % 256 == 0


def test_kv_generate_matches_numpy(lib):
    s = shape(2, 3, 17)
    k = np.zeros((2, 3, 17, 128), np.uint16)
    v = np.zeros_like(k)
    lib.check(lib.kv_generate(None, C.byref(s), 11, 5, A.ptr(k), A.ptr(v)))
    rk, rv = R.gen_kv(2, 3, 17, 128, 11, 5)
    assert np.array_equal(k, rk) and np.array_equal(v, rv)
    assert np.isfinite(R.bf2f(k)).all()


def _kv(L, H, T, seed=3, ctx=1):
    return R.gen_kv(L, H, T, 128, seed, ctx)


def _scores(lib, s, cfg, k):
    out = np.zeros((s.L, s.H, s.T), np.float32)
    lib.check(lib.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(out)))
    return out


def test_knorm_scores_exact(lib):
    s = shape(2, 2, 200)
    k, _ = _kv(2, 2, 200)
    got = _scores(lib, s, plan(lib, "knorm", 0.5, s), k)
    assert np.array_equal(got, R.knorm_scores(k))


def test_keydiff_scores_track_cosine_similarity(lib):
    s = shape(1, 2, 300)
    k, _ = _kv(1, 2, 300)
    got = _scores(lib, s, plan(lib, "keydiff", 0.5, s), k).astype(np.float64)
    sim = R.keydiff_similarity(k)
    # fp32 dot of a unit key with a sum of 300 unit keys: absolute error ~ 1e-7 * T
    np.testing.assert_allclose(-got, sim, rtol=1e-5, atol=1e-7 * 300)


def test_keydiff_scores_exact(lib):
    s = shape(2, 2, 333)
    k, _ = _kv(2, 2, 333)
    got = _scores(lib, s, plan(lib, "keydiff", 0.5, s), k)
    assert np.array_equal(got.view(np.uint32), R.keydiff_scores(k).view(np.uint32))


def test_snapkv_scores_match_numpy(lib):
    s = shape(1, 2, 160)
    k, _ = _kv(1, 2, 160)
    cfg = plan(lib, "snapkv", 0.5, s)
    got = _scores(lib, s, cfg, k)
    q = R.gen_q(1, 2, cfg.q_heads, cfg.window, 128, cfg.q_seed)
    want = R.snapkv_scores(k, q, cfg.window, cfg.q_heads, cfg.pool)
    assert np.array_equal(got.reshape(-1).view(np.uint32), want.reshape(-1).view(np.uint32))


def test_snapkv_caller_queries_match_numpy(lib):
    """Caller-supplied observation-window queries, bf16
    [L][H*G][W][128], replace the synthetic ones: oracle == numpy."""
    s = shape(2, 2, 300)
    k, _ = _kv(2, 2, 300)
    cfg = plan(lib, "snapkv", 0.5, s)
    rng = np.random.default_rng(4)
    qf = rng.standard_normal((2, 2 * cfg.q_heads, cfg.window, 128)).astype(np.float32) * np.float32(9.0)
    q = (qf.view(np.uint32) >> 16).astype(np.uint16)
    out = np.zeros((2, 2, 300), np.float32)
    lib.check(lib.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(q), A.ptr(out)))
    want = R.snapkv_scores(k, q, cfg.window, cfg.q_heads, cfg.pool)
    assert np.array_equal(out.reshape(-1).view(np.uint32), want.reshape(-1).view(np.uint32))
    assert not np.array_equal(out, _scores(lib, s, cfg, k))


def _snap_groups_k(L, H, T, seed=8):
    """Keys that exercise snapkv spec v4's per-16-token K scales: an all-zero
    group (scale 0), a group with one huge outlier row (a large logit factor:
    the clamped E path next to clamp-free blocks), a group of tiny values, a
    constant group, -0, and a ragged last group and block (P = T - 32)."""
    k, _ = _kv(L, H, T, seed=seed)
    x = R.bf2f(k).copy()
    x[:, :, 16:32] = 0.0                                   # group 1: all zero -> tau = 0
    x[:, :, 37] *= np.float32(4e3)                         # group 2: one huge row
    x[:, :, 48:64] *= np.float32(1e-20)                    # group 3: tiny
    x[:, :, 64:80] = np.float32(0.75)                      # group 4: constant
    x[:, :, 81, 3] = np.float32(-0.0)
    x[:, :, 100:108] *= np.float32(-300.0)                 # half of group 6 large and negated
    to_bf = lambda a: (a.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    return to_bf(x)


def _snap_queries(s, cfg, seed=11, spread=3.0):
    rng = np.random.default_rng(seed)
    qf = rng.standard_normal((s.L, s.H * cfg.q_heads, cfg.window, 128)).astype(np.float32) * np.float32(spread)
    return (qf.view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("T", [32 + 300, 32 + 129])
def test_snapkv_k_groups_match_numpy(lib, T):
    """spec v4 K groups (zero, outlier, tiny, constant, ragged): oracle == numpy."""
    s = shape(1, 2, T)
    k = _snap_groups_k(1, 2, T)
    cfg = plan(lib, "snapkv", 0.5, s)
    q = _snap_queries(s, cfg)
    out = np.zeros((1, 2, T), np.float32)
    lib.check(lib.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(q), A.ptr(out)))
    want = R.snapkv_scores(k, q, cfg.window, cfg.q_heads, cfg.pool)
    assert np.array_equal(out.reshape(-1).view(np.uint32), want.reshape(-1).view(np.uint32))


def test_knorm_keep_low_flag(lib):
    s = shape(1, 2, 100)
    k, _ = _kv(1, 2, 100)
    cfg = plan(lib, "knorm", 0.5, s)
    cfg.flags = A.KVT_CODEC_KNORM_KEEP_LOW
    assert np.array_equal(_scores(lib, s, cfg, k), -R.knorm_scores(k))


def test_identity_configuration_has_no_blob(lib):
    """ratio 1.0 at 16 bits keeps every token verbatim: the compressed chunk
    is the source KV (kvt_blob_map.identity), so compress writes nothing and
    unpack refuses. A full keep at fewer bits still quantises."""
    s = shape(1, 2, 64)
    k, v = _kv(1, 2, 64)
    cfg = plan(lib, "knorm", 1.0, s)
    m = A.BlobMap()
    lib.check(lib.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    assert cfg.keep == 64 and cfg.bits == 16 and m.identity == 1 and m.total_bytes == 0
    lib.check(lib.compress(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, None, None))
    with pytest.raises(A.AbiError):
        lib.check(lib.unpack(None, C.byref(s), C.byref(cfg), None, None, None))
    q8 = plan(lib, "knorm-q8", 0.515625, s)  # eff(8) = 8/16 + 1/64: every token at 8 bits
    lib.check(lib.blob_layout(C.byref(s), C.byref(q8), C.byref(m)))
    assert q8.keep == 64 and q8.bits == 8 and m.identity == 0 and m.total_bytes > 0


def test_topk_rule_ties_and_order(lib):
    s = shape(1, 3, 50)
    sc = np.zeros((1, 3, 50), np.float32)
    sc[0, 0] = np.arange(50)[::-1]  # strictly decreasing: keep the first k
    sc[0, 1] = 1.0  # all tied: lowest indices
    sc[0, 1, 40] = 2.0
    sc[0, 2] = np.random.default_rng(1).integers(0, 4, 50)  # heavy ties
    sc[0, 2, 7] = -0.0
    cfg = plan(lib, "knorm", 0.2, s)
    idx = np.zeros((1, 3, cfg.keep), np.int32)
    lib.check(lib.topk(None, C.byref(s), C.byref(cfg), A.ptr(sc), A.ptr(idx)))
    assert idx[0, 0].tolist() == list(range(cfg.keep))
    assert idx[0, 1].tolist() == list(range(cfg.keep - 1)) + [40]
    assert np.array_equal(idx, R.topk_indices(sc, cfg.keep))


def _extreme_kv(L, H, T, seed=5):
    """KV with outliers that defeat the fast quantisation path: huge rows,
    fp16-overflowing groups, tiny ranges far from zero, exact zeros."""
    k, v = _kv(L, H, T, seed=seed)
    rng = np.random.default_rng(seed)
    x = R.bf2f(k).copy()
    y = R.bf2f(v).copy()
    x[:, :, ::7] *= np.float32(3e5)            # whole rows beyond fp16 range
    y[:, :, 1::5] = np.float32(1000.0) + y[:, :, 1::5] * np.float32(1e-3)  # tiny range, large offset
    y[:, :, 2::9] = 0.0
    x[:, :, :, 5] = -x[:, :, :, 5] * np.float32(7e4)
    rr = rng.integers(0, T, size=3)
    x[:, :, rr] = np.float32(-0.0)
    to_bf = lambda a: (a.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)  # truncation is fine: any bf16
    return to_bf(x), to_bf(y)


@pytest.mark.parametrize("bits", [2, 4, 8, 16])
@pytest.mark.parametrize("extreme", [False, True])
def test_pack_matches_numpy_exactly(lib, bits, extreme):
    """The oracle's pack (codes, fp16 params, index copy) == the numpy
    restatement, byte for byte, including groups that need the exact path."""
    s = shape(2, 2, 300)
    k, v = _extreme_kv(2, 2, 300) if extreme else _kv(2, 2, 300)
    cfg = plan(lib, f"knorm-q{bits}" if bits < 16 else "knorm", 0.3 if bits < 16 else 0.5, s)
    cfg.bits = bits
    m = A.BlobMap()
    lib.check(lib.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    rng = np.random.default_rng(bits)
    idx = np.sort(np.stack([np.stack([rng.choice(300, cfg.keep, replace=False) for _ in range(2)]) for _ in range(2)]),
                  axis=-1).astype(np.int32)
    blob = np.zeros(m.total_bytes, np.uint8)
    lib.check(lib.pack(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), A.ptr(idx), A.ptr(blob)))
    want = R.pack_blob(k.reshape(2, 2, 300, 128), v.reshape(2, 2, 300, 128), idx, bits, m)
    assert np.array_equal(blob, want)


@pytest.mark.parametrize("method,ratio", [("knorm-q8", 0.25), ("keydiff-q4", 0.2), ("knorm-q2", 0.1),
                                          ("snapkv", 0.3), ("knorm-q4", 0.05)])
def test_pack_unpack_roundtrip(lib, method, ratio):
    s = shape(2, 2, 300)
    k, v = _kv(2, 2, 300)
    cfg = plan(lib, method, ratio, s)
    m = A.BlobMap()
    lib.check(lib.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    ws = np.zeros(lib.compress_workspace_bytes(C.byref(s), C.byref(cfg)), np.uint8)
    blob = np.zeros(m.total_bytes, np.uint8)
    lib.check(lib.compress(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws), A.ptr(blob)))
    idx = blob[m.idx_off:m.idx_off + m.idx_bytes].view(np.int32).reshape(2, 2, cfg.keep)
    assert (np.diff(idx, axis=-1) > 0).all() and idx.min() >= 0 and idx.max() < 300
    ko = np.zeros((2, 2, cfg.keep, 128), np.uint16)
    vo = np.zeros_like(ko)
    lib.check(lib.unpack(None, C.byref(s), C.byref(cfg), A.ptr(blob), A.ptr(ko), A.ptr(vo)))
    kk = np.take_along_axis(R.bf2f(k), idx[..., None].astype(np.int64), axis=2)
    vv = np.take_along_axis(R.bf2f(v), idx[..., None].astype(np.int64), axis=2)
    if cfg.bits == 16:
        assert np.array_equal(R.bf2f(ko), kk) and np.array_equal(R.bf2f(vo), vv)
        return
    # error bound: half a quantisation step (fp16 scale) plus bf16 output rounding
    b = cfg.bits
    for x, y, axis in ((kk, R.bf2f(ko), 2), (vv, R.bf2f(vo), 3)):
        if axis == 2:  # per channel over groups of 128 kept tokens
            err_ok = True
            for g0 in range(0, cfg.keep, 128):
                seg = x[:, :, g0:g0 + 128]
                step = (seg.max(2, keepdims=True) - seg.min(2, keepdims=True)) / (2 ** b - 1)
                err = np.abs(y[:, :, g0:g0 + 128] - seg)
                err_ok &= bool((err <= 0.51 * step * 1.002 + np.abs(seg) * 2 ** -7 + 1e-3).all())
            assert err_ok
        else:
            step = (x.max(3, keepdims=True) - x.min(3, keepdims=True)) / (2 ** b - 1)
            assert (np.abs(y - x) <= 0.51 * step * 1.002 + np.abs(x) * 2 ** -7 + 1e-3).all()
