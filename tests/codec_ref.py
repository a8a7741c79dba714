"""Independent numpy restatement of the codec spec,
used only to pin the C oracle (tests/test_codec_oracle.py). Written from the
spec, not from oracle/orc_codec.c, in vectorised float64 numpy."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2512_14946_b200 import _abi as A

M64 = (1 << 64) - 1


def mix64(z):
    z = z.astype(np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def synth_bf16(seed, ctx, idx, outlier):
    with np.errstate(over="ignore"):
        base = np.uint64((seed * 0x9E3779B97F4A7C15 + ctx * 0xC2B2AE3D27D4EB4F) & M64)
        z = mix64(base + idx.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    sign = (z & np.uint64(1)).astype(np.uint32)
    mant = ((z >> np.uint64(1)) & np.uint64(0x7F)).astype(np.uint32)
    e = 124 + ((z >> np.uint64(8)) & np.uint64(3)).astype(np.uint32) + np.where(outlier, 3, 0).astype(np.uint32)
    return ((sign << 15) | (e << 7) | mant).astype(np.uint16)


def gen_kv(L, H, T, D, seed, ctx):
    n = L * H * T * D
    i = np.arange(n, dtype=np.uint64)
    d = (i % np.uint64(D)).astype(np.int64)
    k = synth_bf16(seed, ctx, i, d % 16 == 3).reshape(L, H, T, D)
    v = synth_bf16(seed, ctx, i + np.uint64(n), np.zeros(n, bool)).reshape(L, H, T, D)
    return k, v


def bf2f(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def gen_q(L, H, G, W, D, q_seed):
    Hq = H * G
    n = L * Hq * W * D
    i = np.arange(n, dtype=np.uint64)
    d = (i % np.uint64(D)).astype(np.int64)
    return synth_bf16(q_seed, 0x51, i, d % 16 == 3).reshape(L, Hq, W, D)


def knorm_scores(k):
    x = bf2f(k).astype(np.float64)
    return (x * x).sum(-1).astype(np.float32)  # exact in float64 for the synthetic range


def keydiff_similarity(k):
    """mean cosine similarity proxy: khat_t . sum_j khat_j (float64)."""
    x = bf2f(k).astype(np.float64)
    n = np.sqrt((x * x).sum(-1, keepdims=True))
    xn = np.where(n > 0, x / np.where(n > 0, n, 1), 0)
    s = xn.sum(-2, keepdims=True)
    return (xn * s).sum(-1)


def snapkv_scores(k, q, W, G, pool):
    L, H, T, D = k.shape
    P = T - W
    out = np.full((L, H, T), np.inf)
    kf = bf2f(k).astype(np.float64)
    qf = bf2f(q).astype(np.float64)
    for l in range(L):
        for h in range(H):
            rows = qf[l, h * G:(h + 1) * G].reshape(G * W, D)
            lg = rows @ kf[l, h, :P].T / np.sqrt(D)
            p = np.exp(lg - lg.max(1, keepdims=True))
            p /= p.sum(1, keepdims=True)
            vote = p.sum(0)
            pooled = np.array([vote[max(0, t - pool // 2):t + pool // 2 + 1].max() for t in range(P)])
            out[l, h, :P] = pooled
    return out.astype(np.float32)


def topk_indices(scores, k):
    """k largest per row, ties -> lower index, ascending output."""
    S = scores.reshape(-1, scores.shape[-1]).astype(np.float32)
    S = np.where(S == 0, np.float32(0), S)
    out = []
    for row in S:
        order = np.lexsort((np.arange(len(row)), -row.astype(np.float64)))
        out.append(np.sort(order[:k]))
    return np.array(out, np.int32).reshape(scores.shape[:-1] + (k,))
