"""Multi-GPU plumbing of the hot path, one process per GPU.

Per step (bench.py, `RankPlacement`): each rank's profile rows live as one
flat record (kvt_pset_record_pack) in a device send buffer; NCCL
all-gathers the records rank-major (all_gather_into_tensor on the step's
stream) and kvt_pset_merge assembles the global profile set from them on the
device; every rank then runs the identical deterministic greedy over all
contexts and compresses only its own shard.

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

import ctypes as C
from typing import Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import _abi as A
from .kvtier import Engine, MergedPSet, ProfileArrays


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


def pack_record(abi: A.Abi, arrays: ProfileArrays) -> np.ndarray:
    """One rank's profile rows as the flat record of include/kvt_b200.h."""
    g = int(arrays.goff[-1]) if arrays.n else 0
    out = np.zeros(int(abi.pset_record_bytes(arrays.n, g, arrays.M)), np.uint8)
    st = arrays.c_struct()
    abi.check(abi.pset_record_pack(C.byref(st), A.ptr(out)))
    return out


class RankPlacement:
    """The exchange step of one rank: its record in a send buffer on
    `device` (CUDA for NCCL, CPU for gloo), all-gathered into a receive
    buffer and merged into the global profile set by the engine's
    kvt_pset_merge (orc_pset_merge for the CPU restatement). Equal context
    counts and grid lengths on every rank (all_gather_into_tensor)."""

    def __init__(self, eng: Engine, mine: ProfileArrays, group=None, device=None, pin: bool = False,
                 merge_on=None):
        self.eng, self.group = eng, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.n, self.M = mine.n, mine.M
        self.g = int(mine.goff[-1]) if mine.n else 0
        rec = pack_record(eng.abi, mine)
        self.host = torch.from_numpy(rec)
        if pin:
            self.host = self.host.pin_memory()
        dev = torch.device(device) if device is not None else torch.device("cpu")
        self.send = self.host.to(dev).clone() if dev.type == "cuda" else self.host.clone()
        self.recv = torch.empty(self.world * self.send.numel(), dtype=torch.uint8, device=dev)
        self.pset = MergedPSet(eng, self.world * self.n)
        self.h2d_bytes = int(self.send.numel())
        # merge_on: a CUDA device when the collective runs on host buffers
        # (gloo) but the engine merges on the GPU (bench --ranks-share-gpu)
        self.stage = (torch.empty(self.recv.numel(), dtype=torch.uint8, device=merge_on)
                      if merge_on is not None else None)

    def upload(self):
        """Copy the host record into the send buffer (the e2e leg's H2D)."""
        self.send.copy_(self.host, non_blocking=True)

    def exchange(self) -> MergedPSet:
        """All-gather every rank's record, merge on the engine's device."""
        if self.world > 1:
            dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
            src = self.recv
        else:
            src = self.send
        if self.stage is not None:
            self.stage[:src.numel()].copy_(src, non_blocking=True)
            src = self.stage
        return self.pset.merge(src, self.world, self.n, self.g, self.M)
