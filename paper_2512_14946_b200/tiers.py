"""Tier-move executor: applies a placement to bytes.

The reference only models tier moves: a PlacementAction (Insert /
Recompress / Evict, proj/include/kvtier/core.hpp:96-103, built at
proj/src/placement.cpp:213-221) changes occupancy and load-time terms
(SPEC.md:446). Here the GPU tier is HBM (the compressed blob stays where
the codec wrote it), the CPU tier a pinned host arena: moving a context
down copies its blob device -> host, promoting it copies it back, both
through kvt_tier_moves (batched, chunked cudaMemcpyAsync over the handle's
copy streams; the two directions run on different copy engines). The
bottom (SSD) tier is staged through the same pinned arena; the file write
itself is outside the path (storage engine out of scope).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import _abi as A


class HostArena:
    """A pinned host buffer carved into per-context slots (bump allocator)."""

    def __init__(self, abi: A.Abi, nbytes: int):
        self.abi = abi
        p = C.c_void_p()
        abi.check(abi.tier_host_alloc(int(nbytes), C.byref(p)))
        self.base, self.nbytes, self.used = p.value, int(nbytes), 0
        self.slots: Dict[int, Tuple[int, int]] = {}

    def slot(self, ctx: int, nbytes: int) -> int:
        if ctx in self.slots and self.slots[ctx][1] >= nbytes:
            return self.slots[ctx][0]
        off = (self.used + 255) & ~255
        if off + nbytes > self.nbytes:
            raise MemoryError(f"host arena full ({self.nbytes} B)")
        self.used = off + nbytes
        self.slots[ctx] = (self.base + off, nbytes)
        return self.base + off

    def reset(self):
        self.used = 0
        self.slots.clear()

    def close(self):
        if self.base:
            self.abi.tier_host_free(self.base)
            self.base = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TierExecutor:
    """Turns (context, blob, bytes, target tier) into device<->host moves."""

    def __init__(self, eng, arena: HostArena, gpu_tier_index: int = 0):
        self.eng, self.arena, self.gpu = eng, arena, gpu_tier_index

    def moves_for(self, placed: Sequence[Tuple[int, int, int, int]]) -> List[A.Move]:
        """placed = [(ctx, tier_index, device blob address, bytes)]: every
        context below the GPU tier is copied device -> host into its slot."""
        out = []
        for ctx, tier, dptr, nbytes in placed:
            if tier > self.gpu and nbytes > 0:
                out.append(A.Move(dptr, self.arena.slot(ctx, nbytes), int(nbytes), A.KVT_MOVE_D2H, 0))
        return out

    def run(self, moves: Sequence[A.Move]):
        if not moves:
            return
        arr = (A.Move * len(moves))(*moves)
        self.eng.abi.check(self.eng.abi.tier_moves(self.eng.h, arr, len(moves)))

    @staticmethod
    def reverse(moves: Sequence[A.Move]) -> List[A.Move]:
        """The promotion of the same contexts: host slot -> device blob."""
        return [A.Move(m.dst, m.src, m.bytes, A.KVT_MOVE_H2D if m.kind == A.KVT_MOVE_D2H else A.KVT_MOVE_D2H, 0)
                for m in moves]


def host_moves_bytes(moves: Sequence[A.Move]) -> int:
    return int(sum(m.bytes for m in moves))


__all__ = ["HostArena", "TierExecutor", "host_moves_bytes"]
