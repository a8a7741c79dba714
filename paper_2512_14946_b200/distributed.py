"""Multi-GPU plumbing of the hot path, one process per GPU.

KV chunks shard naturally: rank r owns a contiguous range of contexts,
compresses and scores them alone (no cross-context term in
proj/src/utility.cpp:129-145). The one exchange is before the global
greedy: least_drop_update argmins over every resident of a tier
(proj/src/placement.cpp:179-197), so every rank needs every context's
profile. `gather_profiles` all-gathers the per-rank profile rows (a few
hundred bytes per context) with one collective per array; every rank then
runs the identical deterministic greedy over the merged set (replicated,
bit-identical), and compresses only its own contexts.

Backend-agnostic: NCCL on CUDA tensors in bench.py, gloo on CPU tensors in
the multi-process tests. Context ids are rank-prefixed so the merged
byte-lexicographic order (the ABI's context index, ProfileMap order) is
rank-major: rank r's contexts are the index range shard(n_total, world, r).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np
import torch
import torch.distributed as dist

from .kvtier import ProfileArrays


def shard(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of the contexts rank `rank` owns (equal contiguous ranges;
    the last rank takes the remainder)."""
    per = n_total // world
    lo = rank * per
    return lo, (n_total if rank == world - 1 else lo + per)


def context_ids(n_local: int, world: int) -> list:
    """Rank-major ids: byte order == (rank, local index) order."""
    return [f"r{r:03d}-{i:07d}" for r in range(world) for i in range(n_local)]


def merge_rank_profiles(parts) -> ProfileArrays:
    """The global ProfileArrays of per-rank profile sets (equal context count,
    one shared ratio grid): what `gather_profiles` returns on every rank,
    built here from the parts directly (fixtures, single-process checks)."""
    world, n = len(parts), parts[0].n
    G = len(parts[0].grid) // n
    qual = np.concatenate([p.qual.reshape(n, p.M, G) for p in parts])
    return ProfileArrays.uniform_grid(context_ids(n, world), np.concatenate([p.orig for p in parts]),
                                      np.concatenate([p.freq for p in parts]), parts[0].grid[:G], qual,
                                      np.concatenate([p.has for p in parts]))


def gather_profiles(mine: ProfileArrays, group=None, device=None) -> ProfileArrays:
    """All-gather every rank's profile rows into the global ProfileArrays
    (uniform ratio grid, equal context count per rank). `device` is where
    the collective runs: a CUDA device for NCCL, None/CPU for gloo."""
    world = dist.get_world_size(group)
    if world == 1:
        return mine
    n = mine.n
    G = len(mine.grid) // n
    M = mine.M
    dev = torch.device(device) if device is not None else torch.device("cpu")

    def gather(a: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(a)).reshape(-1).to(dev)
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=dev)  # flat: gloo and NCCL agree
        dist.all_gather_into_tensor(out, t, group=group)
        return out.cpu().numpy().reshape((-1,) + tuple(a.shape[1:]))

    orig = gather(mine.orig)
    freq = gather(mine.freq)
    qual = gather(mine.qual.reshape(n, -1)).reshape(world * n, M, G)
    has = gather(mine.has)
    return ProfileArrays.uniform_grid(context_ids(n, world), orig, freq, mine.grid[:G], qual, has)
