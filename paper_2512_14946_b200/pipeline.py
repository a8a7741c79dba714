"""The full hot path for a batch of contexts: score every (context, config,
tier) candidate, run the least-utility-drop greedy over the batch
(insert_joint per context, proj/src/placement.cpp:225-250), then compress
each context's KV chunk with the configuration it was placed at.

Device memory comes from torch (plumbing only); every compute step is a
kvt_* kernel in libkvt_b200.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Tuple

import numpy as np
import torch

from . import _abi as A
from .kvtier import CandidateSpace, Engine, ProfileArrays, PSet, StoreState, UtilityParams


class KVPool:
    """P distinct synthetic KV chunks resident in HBM; context c reads chunk
    c % P (each chunk >> L2, so every read is an HBM read)."""

    def __init__(self, eng: Engine, L: int, H: int, T: int, D: int, n_chunks: int, seed: int = 1):
        self.eng, self.L, self.H, self.T, self.D = eng, L, H, T, D
        n = L * H * T * D
        self.k = [torch.empty(n, dtype=torch.int16, device="cuda") for _ in range(n_chunks)]
        self.v = [torch.empty(n, dtype=torch.int16, device="cuda") for _ in range(n_chunks)]
        s = A.KvShape(L, H, T, D)
        for i in range(n_chunks):
            eng.abi.check(eng.abi.kv_generate(eng.h, C.byref(s), seed, i, A.ptr(self.k[i]), A.ptr(self.v[i])))
        eng.abi.check(eng.abi.sync(eng.h))

    def chunk(self, c: int):
        i = c % len(self.k)
        return self.k[i], self.v[i]


class Codec:
    """Plans and launches compress for (method, ratio, T) configurations.

    With several engines (`lanes`, each a kvt handle on its own CUDA stream
    with its own workspace and output ring), consecutive contexts go to
    different streams so one context's kernels fill the SMs another leaves
    idle (e.g. snapkv's 16-CTA clusters occupy 112 of 148 SMs)."""

    def __init__(self, eng, L: int, H: int, D: int = 128):
        self.lanes = list(eng) if isinstance(eng, (list, tuple)) else [eng]
        self.eng, self.L, self.H, self.D = self.lanes[0], L, H, D
        self._plans: Dict[Tuple[str, float, int], Tuple[A.CodecCfg, A.BlobMap, int]] = {}
        self.ws = None
        self.out: List[torch.Tensor] = []
        self._ws: List[torch.Tensor] = []
        self._out: List[List[torch.Tensor]] = []

    def plan(self, method: str, ratio: float, T: int):
        key = (method, ratio, T)
        p = self._plans.get(key)
        if p is None:
            s = A.KvShape(self.L, self.H, T, self.D)
            cfg = A.CodecCfg()
            self.eng.abi.check(self.eng.abi.codec_plan(method.encode(), ratio, C.byref(s), C.byref(cfg)))
            m = A.BlobMap()
            self.eng.abi.check(self.eng.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
            wsb = self.eng.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg))
            p = (cfg, m, wsb)
            self._plans[key] = p
        return p

    def reserve(self, max_T: int, n_out: int = 2):
        """Workspace + output ring (per lane) for chunks up to max_T tokens."""
        s = A.KvShape(self.L, self.H, max_T, self.D)
        cfg = A.CodecCfg(0, 16, max_T, 32, 4, 7, 0)
        wsb = self.eng.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg))
        m = A.BlobMap()
        self.eng.abi.check(self.eng.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
        self._ws = [torch.empty(wsb, dtype=torch.uint8, device="cuda") for _ in self.lanes]
        self._out = [[torch.empty(m.total_bytes, dtype=torch.uint8, device="cuda") for _ in range(n_out)]
                     for _ in self.lanes]
        self.ws, self.out = self._ws[0], self._out[0]

    def compress(self, method: str, ratio: float, k, v, T: int, slot: int) -> int:
        cfg, m, _ = self.plan(method, ratio, T)
        s = A.KvShape(self.L, self.H, T, self.D)
        li = slot % len(self.lanes)
        eng, outs = self.lanes[li], self._out[li]
        out = outs[(slot // len(self.lanes)) % len(outs)]
        eng.abi.check(eng.abi.compress(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), A.ptr(self._ws[li]),
                                       A.ptr(out)))
        return m.total_bytes

    def launches(self) -> int:
        return sum(int(e.abi.launch_count(e.h)) for e in self.lanes)


def place(store: StoreState, ps: PSet, space: CandidateSpace, params: UtilityParams, order) -> np.ndarray:
    """Empty the store and insert the batch in arrival order."""
    store.clear()
    return store.insert_joint(ps, space, params, order)


def compress_placed(codec: Codec, pool: KVPool, store: StoreState, arrays: ProfileArrays, space: CandidateSpace,
                    bytes_per_token: int) -> Tuple[int, int]:
    """Compress every resident context at its placed (method, ratio)."""
    snap = store.snapshot()
    names = space.method_names
    in_bytes = out_bytes = 0
    for c in range(arrays.n):
        if snap["tier_index"][c] < 0:
            continue
        T = int(arrays.orig[c] // bytes_per_token)
        k, v = pool.chunk(c)
        out_bytes += codec.compress(names[snap["method"][c]], float(snap["ratio"][c]), k, v, T, c)
        in_bytes += int(arrays.orig[c])
    return in_bytes, out_bytes
