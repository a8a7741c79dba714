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


SNAP_C0 = np.float32(0.12751743082459868)  # log2(e) / sqrt(128)
SNAP_P = [np.float32(x) for x in (1.535336188319500E-4, 1.339887440266574E-3, 9.618437357674640E-3,
                                  5.550332471162809E-2, 2.402264791363012E-1, 6.931472028550421E-1)]


def quant_rows_i8(x):
    """int8 codes + fp32 scale per row: absmax/127, rint(x * (127/absmax))."""
    x = x.astype(np.float32)
    a = np.abs(x).max(-1)
    safe = np.where(a > 0, a, np.float32(1))
    inv = (np.float32(127) / safe).astype(np.float32)
    q = np.clip(np.rint((x * inv[..., None]).astype(np.float32)), -127, 127)
    q = np.where(a[..., None] > 0, q, 0).astype(np.int64)
    scale = np.where(a > 0, (a / np.float32(127)).astype(np.float32), np.float32(0))
    return q, scale.astype(np.float32)


def snap_exp_fx(d):
    """round(2^22 * 2^d) for d <= 0 (fp32 mul/add polynomial), 0 below -30."""
    d = d.astype(np.float32)
    n = np.rint(d).astype(np.float32)
    f = (d - n).astype(np.float32)
    p = np.full_like(f, SNAP_P[0])
    for c in SNAP_P[1:] + [np.float32(1.0)]:
        p = (p * f).astype(np.float32)
        p = (p + c).astype(np.float32)
    e = np.clip(n, -30, 0).astype(np.int32)
    x = np.ldexp(p, 22 + e).astype(np.float32)
    return np.where(d < np.float32(-30), 0, np.rint(x)).astype(np.uint64)


def snapkv_scores(k, q, W, G, pool):
    """Exact-integer snapkv, vectorised numpy, float32 ops."""
    L, H, T, D = k.shape
    P = T - W
    out = np.full((L, H, T), np.inf, np.float32)
    if P <= 0:
        return out
    for l in range(L):
        for h in range(H):
            rows = bf2f(q[l, h * G:(h + 1) * G].reshape(G * W, D))
            q8, sig = quant_rows_i8(rows)
            cr = (sig * SNAP_C0).astype(np.float32)
            k8, tau = quant_rows_i8(bf2f(k[l, h, :P]))
            I = q8 @ k8.T  # exact integers
            y = ((I.astype(np.float32) * tau[None, :]).astype(np.float32) * cr[:, None]).astype(np.float32)
            m = y.max(1, keepdims=True)
            E = snap_exp_fx((y - m).astype(np.float32))
            Ls = E.sum(1)
            w = (np.uint64(1) << np.uint64(46)) // Ls
            vote = (E * w[:, None]).sum(0)
            pooled = np.array([vote[max(0, t - pool // 2):t + pool // 2 + 1].max() for t in range(P)], np.uint64)
            out[l, h, :P] = (pooled.astype(np.float64).astype(np.float32) * np.float32(2.0 ** -46)).astype(np.float32)
    return out


def topk_indices(scores, k):
    """k largest per row, ties -> lower index, ascending output."""
    S = scores.reshape(-1, scores.shape[-1]).astype(np.float32)
    S = np.where(S == 0, np.float32(0), S)
    out = []
    for row in S:
        order = np.lexsort((np.arange(len(row)), -row.astype(np.float64)))
        out.append(np.sort(order[:k]))
    return np.array(out, np.int32).reshape(scores.shape[:-1] + (k,))
