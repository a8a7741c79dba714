"""Fidelity of the builder-defined codec spec to the published scorers
(the reference has no codec, so bit parity cannot be pinned to
it; this pins the spec to the algorithms PAPER.md:636-638 names instead).

The exact-integer / fixed-point formulations the CUDA path matches bit for
bit (oracle/orc_codec.c) must keep the same tokens as a
float64 statement of each algorithm on bf16 keys with outlier channels and
a shared per-head offset (as real keys have):
* knorm: squared L2 norm of each key;
* keydiff: minus the cosine of each key to the mean unit key direction;
* snapkv: softmax(q k^T / sqrt(128)) over the prefix for every observation-
  window query of the kv-head's GQA group, summed over the rows, max-pooled
  over +-3 tokens, window tokens always kept.
CPU only: the oracle is bit-identical to the GPU path (tests/test_gpu_codec.py)."""
import ctypes as C

import numpy as np
import pytest

import codec_ref as R
from paper_2512_14946_b200 import _abi as A


def _keys(L, H, T, seed):
    rng = np.random.default_rng(seed)
    kf = rng.standard_normal((L, H, T, 128)).astype(np.float32)
    kf[..., 7] *= np.float32(6.0)
    kf[..., 50] *= np.float32(-4.0)
    kf += rng.standard_normal((L, H, 1, 128)).astype(np.float32) * np.float32(0.5)
    return (kf.view(np.uint32) >> 16).astype(np.uint16)


def _queries(L, H, cfg, seed):
    rng = np.random.default_rng(seed + 100)
    qf = rng.standard_normal((L, H * cfg.q_heads, cfg.window, 128)).astype(np.float32)
    qf[..., 7] *= np.float32(3.0)
    return (qf.view(np.uint32) >> 16).astype(np.uint16)


def _float64_scores(method, k, q, cfg, h):
    x = R.bf2f(k[0, h]).astype(np.float64)
    if method == "knorm":
        return (x * x).sum(1)
    if method == "keydiff":
        u = x / np.linalg.norm(x, axis=1, keepdims=True)
        return -(u @ u.sum(0))
    W, G = cfg.window, cfg.q_heads
    P = x.shape[0] - W
    qq = R.bf2f(q[0, h * G:(h + 1) * G]).astype(np.float64).reshape(G * W, 128)
    lg = qq @ x[:P].T / np.sqrt(128.0)
    p = np.exp(lg - lg.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    v = p.sum(0)
    half = cfg.pool // 2
    pooled = np.array([v[max(0, t - half):t + half + 1].max() for t in range(P)])
    return np.concatenate([pooled, np.full(W, np.inf)])


@pytest.mark.parametrize("method,floor", [("knorm", 0.999), ("keydiff", 0.999), ("snapkv", 0.95)])
@pytest.mark.parametrize("seed", [5, 6])
def test_kept_tokens_match_float64_algorithm(oracle_abi, method, floor, seed):
    lib = oracle_abi
    L, H, T = 1, 4, 2048
    s = A.KvShape(L, H, T, 128)
    cfg = A.CodecCfg()
    lib.check(lib.codec_plan(method.encode(), 0.3, C.byref(s), C.byref(cfg)))
    k = _keys(L, H, T, seed)
    q = _queries(L, H, cfg, seed) if method == "snapkv" else None
    out = np.zeros((L, H, T), np.float32)
    lib.check(lib.token_scores(None, C.byref(s), C.byref(cfg), A.ptr(k), None if q is None else A.ptr(q),
                               A.ptr(out)))
    top = lambda sc: set(np.argsort(-sc, kind="stable")[:cfg.keep].tolist())  # noqa: E731
    for h in range(H):
        overlap = len(top(out[0, h]) & top(_float64_scores(method, k, q, cfg, h))) / cfg.keep
        assert overlap >= floor, (method, h, overlap)
