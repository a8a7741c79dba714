"""Tier-move executor: applies placement actions to bytes.

The reference only models tier moves: the greedy returns a PlacementAction
list (Insert / Recompress / Evict, proj/include/kvtier/core.hpp:96-103, built
at proj/src/placement.cpp:213-221) that changes occupancy and load-time terms
(SPEC.md:446); the paper hands that list to an executor ("RETURN L to
executor"). Here the list drives real byte movement:

* `net_placement` folds a batch's action list, in order, into every
  context's final (tier, method, ratio) — equal to the store snapshot
  (tests/test_tiers.py). Contexts inserted and then recompressed / evicted
  within the same batch are encoded once, at their final configuration.
* GPU tier = HBM: the compressed blob stays where the codec wrote it.
* CPU tier = pinned host DRAM: the blob goes device -> host through
  kvt_tier_moves (chunked cudaMemcpyAsync on the handle's copy streams,
  ordered after the compress on the same stream).
* SSD tier = a file: blobs are staged in pinned DRAM as for the CPU tier and
  written by kvt_tier_file_write (O_DIRECT, worker threads).
* The identity configuration (every token at 16 bits) has no blob: its
  source K and V move instead.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import _abi as A


class HostArena:
    """A pinned host buffer carved into per-context slots (bump allocator);
    slots are 4 KiB aligned so the SSD leg can use O_DIRECT."""

    ALIGN = 4096

    def __init__(self, abi: A.Abi, nbytes: int):
        self.abi = abi
        p = C.c_void_p()
        abi.check(abi.tier_host_alloc(int(nbytes) + self.ALIGN, C.byref(p)))
        self.raw = p.value
        self.base = (self.raw + self.ALIGN - 1) & ~(self.ALIGN - 1)
        self.nbytes, self.used = int(nbytes), 0
        self.slots: Dict[int, Tuple[int, int]] = {}

    def slot(self, ctx: int, nbytes: int) -> int:
        if ctx in self.slots and self.slots[ctx][1] >= nbytes:
            return self.slots[ctx][0]
        off = (self.used + self.ALIGN - 1) & ~(self.ALIGN - 1)
        if off + nbytes > self.nbytes:
            raise MemoryError(f"host arena full ({self.nbytes} B)")
        self.used = off + nbytes
        self.slots[ctx] = (self.base + off, nbytes)
        return self.base + off

    def view(self, addr: int, nbytes: int) -> np.ndarray:
        return np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(addr))

    def reset(self):
        self.used = 0
        self.slots.clear()

    def close(self):
        if self.raw:
            self.abi.tier_host_free(self.raw)
            self.raw = self.base = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StagingRing:
    """R pinned slots of `slot_bytes` each, handed out round-robin: the
    landing zone of device -> host moves whose bytes continue elsewhere (the
    SSD writer) or are only being timed. A slot is rewritten R moves later;
    copies into it are stream-ordered on the handle that issued them."""

    def __init__(self, abi: A.Abi, slot_bytes: int, slots: int = 4):
        self.arena = HostArena(abi, slots * ((slot_bytes + 4095) & ~4095))
        self.slot_bytes = (slot_bytes + 4095) & ~4095
        self.n, self.i = slots, 0

    def next(self, nbytes: int) -> int:
        if nbytes > self.slot_bytes:
            raise MemoryError(f"{nbytes} B does not fit a {self.slot_bytes} B staging slot")
        addr = self.arena.base + self.i * self.slot_bytes
        self.i = (self.i + 1) % self.n
        return addr

    def close(self):
        self.arena.close()


def net_placement(actions: np.ndarray, n_ctx: int, tier_ids: Sequence[int]) -> Dict[str, np.ndarray]:
    """Fold a PlacementAction list (ACTION_DTYPE, in order) into every
    context's final tier index / method / ratio (-1: not placed) and how many
    actions of each kind touched it."""
    tier_index = {int(t): i for i, t in enumerate(tier_ids)}
    out = {"tier_index": np.full(n_ctx, -1, np.int32), "method": np.full(n_ctx, -1, np.int32),
           "ratio": np.zeros(n_ctx, np.float64), "inserts": np.zeros(n_ctx, np.int32),
           "recompress": np.zeros(n_ctx, np.int32), "evicts": np.zeros(n_ctx, np.int32)}
    kinds = {A.KVT_INSERT: "inserts", A.KVT_RECOMPRESS: "recompress", A.KVT_EVICT: "evicts"}
    for a in actions:
        c = int(a["ctx"])
        out["tier_index"][c] = tier_index[int(a["tier_id"])]
        out["method"][c] = int(a["method"])
        out["ratio"][c] = float(a["ratio"])
        out[kinds[int(a["kind"])]][c] += 1
    return out


class SsdTier:
    """The bottom tier as a file (kvt_tier_file_*): pieces of pinned host
    memory written / read at file offsets by worker threads."""

    def __init__(self, abi: A.Abi, path: str, nbytes: int, threads: int = 8):
        self.abi, self.path, self.threads = abi, path, threads
        f = C.c_void_p()
        abi.check(abi.tier_file_open(path.encode(), int(nbytes), C.byref(f)))
        self.f = f
        self.direct = bool(abi.tier_file_direct(f))
        self.nbytes, self.used = int(nbytes), 0

    def alloc(self, nbytes: int) -> int:
        off = (self.used + 4095) & ~4095
        if off + nbytes > self.nbytes:
            raise MemoryError("ssd tier file full")
        self.used = off + nbytes
        return off

    def _io(self, fn, pieces):
        arr = (A.FileIo * len(pieces))(*[A.FileIo(h, int(n), int(o)) for h, n, o in pieces])
        self.abi.check(fn(self.f, arr, len(pieces), self.threads))

    def write(self, pieces: Sequence[Tuple[int, int, int]]):
        """pieces = [(host address, bytes, file offset)]"""
        self._io(self.abi.tier_file_write, pieces)

    def read(self, pieces: Sequence[Tuple[int, int, int]]):
        self._io(self.abi.tier_file_read, pieces)

    def close(self, remove: bool = True):
        if self.f:
            self.abi.tier_file_close(self.f)
            self.f = None
            if remove:
                try:
                    os.unlink(self.path)
                except OSError:
                    pass

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TierExecutor:
    """Enqueues the device -> host leg of contexts placed below the GPU tier
    on the engine (handle) whose stream produced their bytes."""

    def __init__(self, eng, arena, gpu_tier_index: int = 0):
        self.eng, self.arena, self.gpu = eng, arena, gpu_tier_index

    def moves_for(self, placed: Sequence[Tuple[int, int, int, int]]) -> List[A.Move]:
        """placed = [(ctx, tier_index, device address, bytes)]: every context
        below the GPU tier is copied device -> host into its arena slot."""
        out = []
        for ctx, tier, dptr, nbytes in placed:
            if tier > self.gpu and nbytes > 0:
                out.append(A.Move(dptr, self.arena.slot(ctx, nbytes), int(nbytes), A.KVT_MOVE_D2H, 0))
        return out

    def run(self, moves: Sequence[A.Move], eng=None):
        if not moves:
            return
        eng = eng or self.eng
        arr = (A.Move * len(moves))(*moves)
        eng.abi.check(eng.abi.tier_moves(eng.h, arr, len(moves)))

    @staticmethod
    def reverse(moves: Sequence[A.Move]) -> List[A.Move]:
        """The promotion of the same contexts: host slot -> device blob."""
        return [A.Move(m.dst, m.src, m.bytes, A.KVT_MOVE_H2D if m.kind == A.KVT_MOVE_D2H else A.KVT_MOVE_D2H, 0)
                for m in moves]


def context_sources(blob_addr: int, m: A.BlobMap, k_addr: int, v_addr: int, kv_bytes: int) -> List[Tuple[int, int]]:
    """The device ranges that hold a compressed context: its blob, or for the
    identity configuration the source K and V it aliases."""
    if m.identity:
        return [(k_addr, kv_bytes), (v_addr, kv_bytes)]
    return [(blob_addr, int(m.total_bytes))]


def host_moves_bytes(moves: Sequence[A.Move]) -> int:
    return int(sum(m.bytes for m in moves))


__all__ = ["HostArena", "StagingRing", "SsdTier", "TierExecutor", "net_placement", "context_sources",
           "host_moves_bytes"]
