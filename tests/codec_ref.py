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


def row_dot32(x, y):
    """Canonical fp32 row dot product: per 8-channel chunk an
    even- and an odd-channel fma chain, chunk = even + odd, then a butterfly
    over the 16 chunk sums (strides 8, 4, 2, 1)."""
    x = x.astype(np.float32)
    y = np.broadcast_to(y.astype(np.float32), x.shape)
    sh = x.shape[:-1] + (16, 8)
    xc, yc = x.reshape(sh), y.reshape(sh)
    e = np.zeros(sh[:-1], np.float32)
    o = np.zeros(sh[:-1], np.float32)
    for q in range(4):
        e = fma32(xc[..., 2 * q], yc[..., 2 * q], e)
        o = fma32(xc[..., 2 * q + 1], yc[..., 2 * q + 1], o)
    p = (e + o).astype(np.float32)
    idx = np.arange(16)
    for off in (8, 4, 2, 1):
        p = (p + p[..., idx ^ off]).astype(np.float32)
    return p[..., 0]


def knorm_scores(k):
    x = bf2f(k)
    return row_dot32(x, x)


def keydiff_scores(k):
    """Exact keydiff v2: inverse norms 1/sqrt(n2) (two RN fp32
    ops, 0 below 2^-100), unit components rounded to 2^-21 fixed point and
    summed in int64, then -(dot(x, S * 2^-21) * inv)."""
    x = bf2f(k)
    n2 = row_dot32(x, x)
    ok = n2 >= np.float32(2.0 ** -100)
    inv = np.where(ok, (np.float32(1) / np.sqrt(np.where(ok, n2, 1)).astype(np.float32)).astype(np.float32), 0)
    inv = inv.astype(np.float32)
    c = (inv * np.float32(2.0 ** 21)).astype(np.float32)
    f = np.rint(x.astype(np.float64) * c[..., None].astype(np.float64)).astype(np.int64)  # exact product
    S = f.sum(-2, keepdims=True)
    sd = (S.astype(np.float32) * np.float32(2.0 ** -21)).astype(np.float32)
    return (-(row_dot32(x, sd) * inv).astype(np.float32)).astype(np.float32)


def keydiff_similarity(k):
    """mean cosine similarity proxy: khat_t . sum_j khat_j (float64)."""
    x = bf2f(k).astype(np.float64)
    n = np.sqrt((x * x).sum(-1, keepdims=True))
    xn = np.where(n > 0, x / np.where(n > 0, n, 1), 0)
    s = xn.sum(-2, keepdims=True)
    return (xn * s).sum(-1)


SNAP_C0 = np.float32(0.12751743082459868)  # log2(e) / sqrt(128)
SNAP_E = [np.float32(float.fromhex(x)) for x in ("0x1.ffec2ep+6", "0x1.683ef2p+6", "0x1.f22ab4p+4")]
# 2^7 * 2^f on [-1/2, 1/2], degree 2 (spec v3)
SNAP_LSH = 24  # block sums scaled by 2^24 in the row sum
SNAP_KGRP = 16  # tokens per K int8 scale (spec v4)
SNAP_AMAX = np.float32(0.25)  # cap of the logit factor a (spec v4)
SNAP_VOTE_SCALE = np.float32(2.0 ** -37)


def fma32(a, b, c):
    """Correctly rounded float32 a*b+c (IEEE fusedMultiplyAdd), vectorised.
    a*b is exact in float64; s = fl64(ab + c) is off the exact sum by err
    (TwoSum, exact). Rounding s to float32 is correct unless s sits exactly
    on a float32 midpoint, where the sign of err breaks the tie."""
    a, b, c = (np.asarray(x, np.float32).astype(np.float64) for x in (a, b, c))
    ab = a * b
    s = ab + c
    bb = s - ab
    err = (ab - (s - bb)) + (c - bb)
    r = s.astype(np.float32)
    lo = np.nextafter(r, np.float32(-np.inf)).astype(np.float64)
    hi = np.nextafter(r, np.float32(np.inf)).astype(np.float64)
    rd = r.astype(np.float64)
    # s exactly halfway between r and a neighbour: the exact value decides
    up = (s == (rd + hi) / 2) & (err > 0)  # exact value just above the upper midpoint
    dn = (s == (rd + lo) / 2) & (err < 0)  # exact value just below the lower midpoint
    r = np.where(up, hi.astype(np.float32), r)
    r = np.where(dn, lo.astype(np.float32), r)
    return r.astype(np.float32)


def quant_i8(x, axis):
    """int8 codes + fp32 scale: absmax/127 over `axis`, rint(x * (127/absmax))."""
    x = x.astype(np.float32)
    a = np.abs(x).max(axis=axis, keepdims=True)
    safe = np.where(a > 0, a, np.float32(1))
    inv = (np.float32(127) / safe).astype(np.float32)
    q = np.clip(np.rint(x.astype(np.float64) * inv.astype(np.float64)), -127, 127)  # rint of the exact product
    q = np.where(a > 0, q, 0).astype(np.int64)
    scale = np.where(a > 0, (a / np.float32(127)).astype(np.float32), np.float32(0))
    return q, scale.astype(np.float32)


def snap_exp_u8(d):
    """round(2^7 * 2^max(d, -16)) with the fixed fp32 FMA polynomial (v3)."""
    d = np.asarray(d, np.float32)
    dc = np.maximum(d, np.float32(-16))
    t = (dc + np.float32(12582912)).astype(np.float32)
    n = (t - np.float32(12582912)).astype(np.float32)
    f = (dc - n).astype(np.float32)
    p = fma32(SNAP_E[2], f, SNAP_E[1])
    p = fma32(p, f, SNAP_E[0])
    x = (p.view(np.uint32) + (t.view(np.uint32) << np.uint32(23))).astype(np.uint32).view(np.float32)
    return ((x + np.float32(8388608)).astype(np.float32).view(np.uint32) - np.uint32(0x4B000000)).astype(np.uint64)


def snapkv_scores(k, q, W, G, pool):
    """Exact-integer snapkv v4, vectorised numpy, float32 ops."""
    L, H, T, D = k.shape
    P = T - W
    out = np.full((L, H, T), np.inf, np.float32)
    if P <= 0:
        return out
    nblk = (P + 31) // 32
    for l in range(L):
        for h in range(H):
            rows = bf2f(q[l, h * G:(h + 1) * G].reshape(G * W, D))
            q8, sig = quant_i8(rows, 1)
            sig = sig[:, 0]
            kx = bf2f(k[l, h, :P])
            k8 = np.zeros((P, D), np.int64)
            tau = np.zeros(P, np.float32)
            for t0 in range(0, P, SNAP_KGRP):  # spec v4: one K scale per 16-token group
                c, sc = quant_i8(kx[t0:t0 + SNAP_KGRP], None)
                k8[t0:t0 + SNAP_KGRP] = c
                tau[t0:t0 + SNAP_KGRP] = sc.reshape(())
            I = q8 @ k8.T  # exact integers [R, P]
            a = ((tau[None, :] * sig[:, None]).astype(np.float32) * SNAP_C0).astype(np.float32)  # per (r, t)
            a = np.minimum(a, SNAP_AMAX)  # v4 cap: keeps -M - 12582912 a exact
            a = (a.view(np.uint32) & np.uint32(0xFFFFFFFC)).view(np.float32)  # 22-bit mantissa: exact offsets
            blk = np.arange(P) // 32
            y = (I.astype(np.float32) * a).astype(np.float32)  # fl(I * a): monotone in I for one group's a
            ypad = np.full((G * W, nblk * 32), -np.inf, np.float32)
            ypad[:, :P] = y
            M = np.ceil(ypad.reshape(G * W, nblk, 32).max(-1)).astype(np.int64)  # ceil of the block's largest fl(I a)
            cb = ((-M[:, blk]).astype(np.float32) - (np.float32(12582912) * a).astype(np.float32)).astype(np.float32)
            X = ((I + 0x4B400000).astype(np.uint32)).view(np.float32)
            E = snap_exp_u8(fma32(X, a, cb))
            Lb = np.add.reduceat(E, np.arange(0, P, 32), axis=1).astype(np.uint64)
            m = M.max(1, keepdims=True)
            sh = (m - M)
            Lr = np.where(sh < 64, (Lb << np.uint64(SNAP_LSH)) >> np.minimum(sh, 63).astype(np.uint64), 0).sum(1)
            Wt = np.where(Lr > 0, (np.uint64(1) << np.uint64(61)) // np.maximum(Lr, 1), 0).astype(np.uint64)
            Wb = np.where(sh < 64, Wt[:, None] >> np.minimum(sh, 63).astype(np.uint64), 0).astype(np.uint64)
            vote = (E * Wb[:, blk]).sum(0)
            pooled = np.array([vote[max(0, t - pool // 2):t + pool // 2 + 1].max() for t in range(P)], np.uint64)
            out[l, h, :P] = (pooled.astype(np.float64).astype(np.float32) * SNAP_VOTE_SCALE).astype(np.float32)
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


def _params(mn, mx, bits):
    """make_param: fp16 scale (max-min)/levels and zero = min."""
    mn = (mn.astype(np.float32) + np.float32(0)).astype(np.float32)  # -0 -> +0
    mx = (mx.astype(np.float32) + np.float32(0)).astype(np.float32)
    levels = np.float32((1 << bits) - 1)
    with np.errstate(over="ignore", invalid="ignore"):
        scale = ((mx - mn) / levels).astype(np.float32)
        s16 = scale.astype(np.float16)
        z16 = mn.astype(np.float16)
        sf = s16.astype(np.float32)
        inv = np.where(sf > 0, (np.float32(1) / np.where(sf > 0, sf, 1)).astype(np.float32), np.float32(0))
    return s16, z16, z16.astype(np.float32), inv.astype(np.float32)


def _codes(x, zf, inv, bits):
    """clamp(rint(exact((x - zf) * inv)), 0, 2^b - 1); NaN -> 0."""
    with np.errstate(over="ignore", invalid="ignore"):
        d = (x.astype(np.float32) - zf).astype(np.float32)
        r = np.rint(d.astype(np.float64) * inv.astype(np.float64))
        r = np.where(r >= 0, np.minimum(r, (1 << bits) - 1), 0)
    return r.astype(np.uint32)


def _pack_words(codes, bits):
    """codes [..., 128] -> u32 words, code of channel d at bit b * (d % (32 / b))."""
    per = 32 // bits
    c = codes.reshape(codes.shape[:-1] + (128 // per, per)).astype(np.uint64)
    sh = (np.arange(per, dtype=np.uint64) * np.uint64(bits))
    return (c << sh).sum(-1).astype(np.uint32)


def pack_blob(k, v, idx, bits, m):
    """Exact numpy restatement of pack (K per channel over groups of 128 kept
    tokens, V per kept token), returned as the blob byte array for layout m."""
    L, H, T, D = k.shape
    keep = idx.shape[-1]
    blob = np.zeros(m.total_bytes, np.uint8)
    blob[m.idx_off:m.idx_off + m.idx_bytes] = idx.astype(np.int32).reshape(-1).view(np.uint8)
    kx = np.take_along_axis(bf2f(k), idx[..., None].astype(np.int64), axis=2)  # [L,H,keep,D]
    vx = np.take_along_axis(bf2f(v), idx[..., None].astype(np.int64), axis=2)
    if bits == 16:
        blob[m.kcode_off:m.kcode_off + m.kcode_bytes] = np.take_along_axis(
            k, idx[..., None].astype(np.int64), axis=2).reshape(-1).view(np.uint8)
        blob[m.vcode_off:m.vcode_off + m.vcode_bytes] = np.take_along_axis(
            v, idx[..., None].astype(np.int64), axis=2).reshape(-1).view(np.uint8)
        return blob
    ng = (keep + 127) // 128
    kc = np.zeros((L, H, keep, 128 * bits // 32), np.uint32)
    ks = np.zeros((L, H, ng, D), np.float16)
    kz = np.zeros((L, H, ng, D), np.float16)
    for g in range(ng):
        seg = kx[:, :, g * 128:(g + 1) * 128]
        s16, z16, zf, inv = _params(seg.min(2), seg.max(2), bits)
        ks[:, :, g], kz[:, :, g] = s16, z16
        kc[:, :, g * 128:(g + 1) * 128] = _pack_words(_codes(seg, zf[:, :, None], inv[:, :, None], bits), bits)
    vs16, vz16, vzf, vinv = _params(vx.min(3), vx.max(3), bits)
    vc = _pack_words(_codes(vx, vzf[..., None], vinv[..., None], bits), bits)
    for off, arr in ((m.kcode_off, kc), (m.kscale_off, ks), (m.kzero_off, kz), (m.vcode_off, vc),
                     (m.vscale_off, vs16), (m.vzero_off, vz16)):
        b = arr.reshape(-1).view(np.uint8)
        blob[off:off + b.size] = b
    return blob
