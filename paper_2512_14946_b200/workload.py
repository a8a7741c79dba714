"""Synthetic inputs for the BASELINE configs. Not an oracle:
these are the *inputs* both arms (CUDA and reference) consume.

Profiles follow the reference's generator conventions: sensitivity-anchored
curves (synth_quality, proj/src/quality.cpp:115-127) applied to the kept
token fraction plus a per-bit-width quantisation cost, one shared grid, and
Zipf-shaped frequencies (assign_zipf_frequencies, proj/src/workload.cpp:
236-245, arrival rate 4, exponent 1). With these tables the greedy places a
mix of q4 / q8 / token-drop / uncompressed configurations (c2, 1000 ctx:
~19 % at ratio 1.0), so the codec does real work. KV chunks come from the counter hash
of the codec spec (kvt_kv_generate), so no dataset is needed.
"""
from __future__ import annotations

import numpy as np

from .kvtier import CandidateSpace, ProfileArrays, TierSpec, UtilityParams

LLAMA8B = dict(L=32, H=8, D=128)   # Llama-3.1-8B / Mistral-7B KV: 131,072 B/token
LLAMA70B = dict(L=80, H=8, D=128)  # 327,680 B/token

QUANT_TOKEN_DROP_METHODS = ["keydiff", "knorm", "snapkv", "keydiff-q8", "knorm-q8", "snapkv-q8",
                            "keydiff-q4", "knorm-q4", "snapkv-q4"]
MIXED_BITS_METHODS = ["keydiff-q8", "knorm-q4", "snapkv-q2", "knorm-q2", "keydiff-q4", "snapkv-q8"]
C5_METHODS = ["keydiff", "knorm-q4", "snapkv-q8"]
DEFAULT_GRID = [0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 1.0]


def bytes_per_token(L, H, D, **_):
    return L * H * D * 2 * 2  # K and V, bf16


def three_tiers(total_bytes, gpu_frac=0.10, cpu_frac=0.30):
    """gpu `gpu_frac` of bytes @8e12 B/s, cpu `cpu_frac` @5e10, ssd unlimited @6e9 + 1e-4 s."""
    return [TierSpec(0, "gpu", int(total_bytes * gpu_frac), 8e12, 0.0),
            TierSpec(1, "cpu", int(total_bytes * cpu_frac), 5e10, 0.0),
            TierSpec(2, "ssd", None, 6e9, 1e-4)]


QUANT_LOSS = {8: 0.002, 4: 0.01, 2: 0.04}  # quality cost of b-bit codes per unit sensitivity


def eff_bytes(bits):
    """Retained bytes per bf16 byte of a b-bit blob (codes + fp16 params);
    DESIGN.md §4.1, same arithmetic as kvt_codec_plan."""
    return 1.0 if bits >= 16 else bits / 16.0 + 1.0 / 64.0


def codec_bits_keep(method, ratio):
    """(bits, kept token fraction) the codec uses for `ratio` (kvt_codec_plan)."""
    b = int(method.split("-q")[1]) if "-q" in method else 16
    bb = next(w for w in (2, 4, 8, 16) if w >= b and (w == 16 or ratio <= eff_bytes(w)))
    return bb, min(1.0, ratio / eff_bytes(bb))


def profiles(n_ctx, space: CandidateSpace, seed=7, tokens=8192, bpt=131072, varied=False,
             sensitivity=(0.0, 0.05), shape_k=1.5) -> ProfileArrays:
    """Synthetic quality tables for "<scorer>[-q<b>]" methods. Token dropping
    follows the reference's curve synth_quality (proj/src/quality.cpp:115-127),
    1 - s*((1 - keep)/0.1)^k, applied to the fraction of tokens the codec
    keeps at that ratio; b-bit codes cost QUANT_LOSS[b] x U(0.5, 1.5) more.
    One sensitivity per (context, scorer), uniform in `sensitivity`."""
    rng = np.random.default_rng(seed)
    M = len(space.methods)
    grid = sorted(space.ratios)
    if varied:
        orig = (rng.integers(1024, 2 * tokens, size=n_ctx) * bpt).astype(np.int64)
    else:
        orig = np.full(n_ctx, tokens * bpt, np.int64)
    scorers = ["keydiff", "knorm", "snapkv"]
    s = rng.uniform(*sensitivity, size=(n_ctx, len(scorers)))
    u = rng.uniform(0.5, 1.5, size=(n_ctx, len(scorers)))
    q = np.zeros((n_ctx, M, len(grid)))
    for m, meth in enumerate(space.methods):
        sc = scorers.index(meth.name.split("-")[0])
        for gi, r in enumerate(grid):
            bits, keep = codec_bits_keep(meth.name, r)
            drop = s[:, sc] * ((1.0 - keep) / 0.1) ** shape_k
            qloss = 0.0 if bits == 16 else QUANT_LOSS[bits] * u[:, sc]
            q[:, m, gi] = np.clip(1.0 - drop - qloss, 0.0, 1.0)
    ranks = rng.permutation(n_ctx)
    w = 1.0 / (ranks + 1.0)
    freq = 4.0 * w / w.sum()
    ids = [f"ctx-{i:07d}" for i in range(n_ctx)]
    return ProfileArrays.uniform_grid(ids, orig, freq, grid, q)


CONFIGS = {
    # configs[0]: the CPU reference's smallest case
    "c1": dict(model="llama-3.1-8b", n_ctx=64, tokens=4096, methods=["keydiff", "knorm", "snapkv"],
               gpu_frac=0.10, varied=False),
    # configs[1]: the headline single-GPU workload
    "c2": dict(model="llama-3.1-8b", n_ctx=1000, tokens=8192, methods=QUANT_TOKEN_DROP_METHODS,
               gpu_frac=0.10, varied=False),
    # configs[2]: Mistral-7B KV, mixed 2/4/8-bit, tight GPU tier
    "c3": dict(model="mistral-7b", n_ctx=1000, tokens=8192, methods=MIXED_BITS_METHODS,
               gpu_frac=0.03, varied=True),
    # configs[3]: Llama-3.1-70B-shaped KV, 10K contexts (sharded)
    "c4": dict(model="llama-3.1-70b", n_ctx=10000, tokens=8192, methods=["keydiff", "knorm", "snapkv"],
               gpu_frac=0.10, varied=False),
    # configs[4]: 1M chunk-config candidates (13,889 x 72); one token-drop, one
    # q4 and one q8 method so the pass exercises quantise/pack as well
    "c5": dict(model="llama-3.1-8b", n_ctx=13889, tokens=8192, methods=C5_METHODS,
               gpu_frac=0.10, varied=True),
}


def build(name, n_ctx=None, seed=7):
    c = dict(CONFIGS[name])
    if n_ctx is not None:
        c["n_ctx"] = n_ctx
    shape = LLAMA70B if c["model"] == "llama-3.1-70b" else LLAMA8B
    space = CandidateSpace(c["methods"], DEFAULT_GRID)
    bpt = bytes_per_token(**shape)
    arr = profiles(c["n_ctx"], space, seed=seed, tokens=c["tokens"], bpt=bpt, varied=c["varied"])
    tiers = three_tiers(int(arr.orig.sum()), c["gpu_frac"], 0.30)
    return dict(cfg=c, shape=shape, space=space, arrays=arr, tiers=tiers, params=UtilityParams(alpha=1.0),
                bytes_per_token=bpt)
