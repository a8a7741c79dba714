"""ctypes mirror of include/kvt_b200.h.

The same ABI is implemented three times (kvt_ = CUDA product, orc_ = CPU
oracle, ref_ = the reference library); `Abi(path, prefix)` binds any of them
so one set of numpy inputs can be pushed through all three.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

KVT_OK, KVT_EVALIDATION, KVT_ETRACE, KVT_ECUDA, KVT_EINVAL, KVT_ENOMEM = range(6)
KVT_INSERT, KVT_RECOMPRESS, KVT_EVICT = range(3)
KVT_RULE_UTILITY, KVT_RULE_QUALITY_FIRST = range(2)
KVT_SCORER_KNORM, KVT_SCORER_KEYDIFF, KVT_SCORER_SNAPKV = range(3)
MAX_TIERS, MAX_METHODS, MAX_RATIOS = 8, 16, 32
QGROUP = 128


class Tier(C.Structure):
    _fields_ = [("tier_id", C.c_int32), ("unlimited", C.c_int32), ("capacity_bytes", C.c_int64),
                ("read_bandwidth", C.c_double), ("fixed_access_latency", C.c_double)]


class Space(C.Structure):
    _fields_ = [("n_methods", C.c_int32), ("method_names", C.POINTER(C.c_char_p)),
                ("decompression_overhead", C.POINTER(C.c_double)), ("n_ratios", C.c_int32),
                ("ratios", C.POINTER(C.c_double))]


class Params(C.Structure):
    _fields_ = [("alpha", C.c_double)]


class Profiles(C.Structure):
    _fields_ = [("n_ctx", C.c_int32), ("n_methods", C.c_int32),
                ("original_size_bytes", C.POINTER(C.c_int64)), ("frequency", C.POINTER(C.c_double)),
                ("grid_offset", C.POINTER(C.c_int32)), ("grid", C.POINTER(C.c_double)),
                ("quality", C.POINTER(C.c_double)), ("has_method", C.POINTER(C.c_uint8))]


class Action(C.Structure):
    _fields_ = [("kind", C.c_int32), ("ctx", C.c_int32), ("tier_id", C.c_int32),
                ("method", C.c_int32), ("ratio", C.c_double)]


class Update(C.Structure):
    _fields_ = [("ctx", C.c_int32), ("kind", C.c_int32), ("tier_index", C.c_int32),
                ("tier_id", C.c_int32), ("method", C.c_int32), ("pad_", C.c_int32),
                ("ratio", C.c_double), ("size_bytes", C.c_int64), ("quality", C.c_double),
                ("ttft", C.c_double), ("utility", C.c_double), ("utility_drop", C.c_double),
                ("bytes_freed", C.c_int64)]


class Best(C.Structure):
    _fields_ = [("status", C.c_int32), ("tier_index", C.c_int32), ("tier_id", C.c_int32),
                ("method", C.c_int32), ("ratio_index", C.c_int32), ("pad_", C.c_int32),
                ("ratio", C.c_double), ("size_bytes", C.c_int64), ("quality", C.c_double),
                ("ttft", C.c_double), ("utility", C.c_double)]


class Entry(C.Structure):
    _fields_ = [("tier_index", C.c_int32), ("method", C.c_int32), ("ratio", C.c_double),
                ("original_size_bytes", C.c_int64), ("frequency", C.c_int64),
                ("last_access", C.c_int64), ("seq", C.c_int64)]


class KvShape(C.Structure):
    _fields_ = [("L", C.c_int32), ("H", C.c_int32), ("T", C.c_int32), ("D", C.c_int32)]


KVT_CODEC_KNORM_KEEP_LOW = 1


class CodecCfg(C.Structure):
    _fields_ = [("scorer", C.c_int32), ("bits", C.c_int32), ("keep", C.c_int32),
                ("window", C.c_int32), ("q_heads", C.c_int32), ("pool", C.c_int32),
                ("flags", C.c_int32), ("pad_", C.c_int32), ("q_seed", C.c_uint64)]


class BlobMap(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "idx_off", "idx_bytes", "kcode_off", "kcode_bytes", "kscale_off", "kzero_off",
        "kparam_bytes", "vcode_off", "vcode_bytes", "vscale_off", "vzero_off", "vparam_bytes",
        "total_bytes", "identity")]


class Move(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("bytes", C.c_int64), ("kind", C.c_int32),
                ("pad_", C.c_int32)]


KVT_MOVE_D2H, KVT_MOVE_H2D, KVT_MOVE_D2D, KVT_MOVE_H2H = 0, 1, 2, 3


class FileIo(C.Structure):
    _fields_ = [("host", C.c_void_p), ("bytes", C.c_int64), ("offset", C.c_int64)]

ACTION_DTYPE = np.dtype([("kind", "<i4"), ("ctx", "<i4"), ("tier_id", "<i4"), ("method", "<i4"),
                         ("ratio", "<f8")])
ENTRY_DTYPE = np.dtype([("tier_index", "<i4"), ("method", "<i4"), ("ratio", "<f8"),
                        ("original_size_bytes", "<i8"), ("frequency", "<i8"),
                        ("last_access", "<i8"), ("seq", "<i8")])
BEST_DTYPE = np.dtype([("status", "<i4"), ("tier_index", "<i4"), ("tier_id", "<i4"),
                       ("method", "<i4"), ("ratio_index", "<i4"), ("pad_", "<i4"),
                       ("ratio", "<f8"), ("size_bytes", "<i8"), ("quality", "<f8"),
                       ("ttft", "<f8"), ("utility", "<f8")])
assert ACTION_DTYPE.itemsize == C.sizeof(Action)
assert ENTRY_DTYPE.itemsize == C.sizeof(Entry)
assert BEST_DTYPE.itemsize == C.sizeof(Best)

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
i32, i64, f64, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64

PLACEMENT_SIGS = {
    "last_error": (C.c_char_p, []),
    "abi_version": (C.c_int, []),
    "create": (C.c_int, [C.c_int, P, PP]),
    "destroy": (C.c_int, [P]),
    "pset_create": (C.c_int, [P, C.POINTER(Profiles), PP]),
    "pset_destroy": (C.c_int, [P]),
    "score_candidates": (C.c_int, [P, P, C.POINTER(Tier), i32, C.POINTER(Space), C.POINTER(Params),
                                   P, P, P, P, P]),
    "best_config": (C.c_int, [P, P, C.POINTER(Tier), i32, C.POINTER(Space), C.POINTER(Params), i32, P]),
    "store_create": (C.c_int, [P, C.POINTER(Tier), i32, i32, PP]),
    "store_destroy": (C.c_int, [P]),
    "store_bind_space": (C.c_int, [P, C.POINTER(Space)]),
    "store_add": (C.c_int, [P, i32, C.POINTER(Entry)]),
    "store_remove": (C.c_int, [P, i32, C.POINTER(Entry)]),
    "store_reconfigure": (C.c_int, [P, i32, i32, f64]),
    "store_touch": (C.c_int, [P, i32, i64]),
    "store_touch_many": (C.c_int, [P, P, P, i64]),
    "store_clear": (C.c_int, [P]),
    "store_occupancy": (C.c_int, [P, P]),
    "store_snapshot": (C.c_int, [P, P]),
    "least_drop_update": (C.c_int, [P, P, C.POINTER(Space), C.POINTER(Params), i32, C.POINTER(Update)]),
    "resolve_overflow": (C.c_int, [P, P, C.POINTER(Space), C.POINTER(Params), C.POINTER(i64)]),
    "insert_joint": (C.c_int, [P, P, C.POINTER(Space), C.POINTER(Params), i32, P, P, P, i64,
                               C.POINTER(i64), C.POINTER(i64)]),
    "rearrange": (C.c_int, [P, P, C.POINTER(Space), C.POINTER(Params), i32, C.POINTER(i64)]),
    "store_actions": (C.c_int, [P, P, i64]),
    "placement_utility": (C.c_int, [P, P, C.POINTER(Space), C.POINTER(Params), C.POINTER(f64)]),
}

CODEC_SIGS = {
    "codec_plan": (C.c_int, [C.c_char_p, f64, C.POINTER(KvShape), C.POINTER(CodecCfg)]),
    "blob_layout": (C.c_int, [C.POINTER(KvShape), C.POINTER(CodecCfg), C.POINTER(BlobMap)]),
    "kv_generate": (C.c_int, [P, C.POINTER(KvShape), u64, u64, P, P]),
    "token_scores": (C.c_int, [P, C.POINTER(KvShape), C.POINTER(CodecCfg), P, P, P]),
    "topk": (C.c_int, [P, C.POINTER(KvShape), C.POINTER(CodecCfg), P, P]),
    "pack": (C.c_int, [P, C.POINTER(KvShape), C.POINTER(CodecCfg), P, P, P, P]),
    "unpack": (C.c_int, [P, C.POINTER(KvShape), C.POINTER(CodecCfg), P, P, P]),
    "compress": (C.c_int, [P, C.POINTER(KvShape), C.POINTER(CodecCfg), P, P, P, P, P]),
    "compress_workspace_bytes": (i64, [C.POINTER(KvShape), C.POINTER(CodecCfg)]),
}

PRODUCT_EXTRA_SIGS = {
    "sync": (C.c_int, [P]),
    "set_stream": (C.c_int, [P, P]),
    "launch_count": (i64, [P]),
    "tier_host_alloc": (C.c_int, [i64, PP]),
    "tier_host_free": (C.c_int, [P]),
    "compress_slices": (C.c_int, [P, C.POINTER(KvShape), C.POINTER(CodecCfg), P, P, i32, i32, P, P]),
}
TIER_SIGS = {"tier_moves": (C.c_int, [P, C.POINTER(Move), i64])}
FILE_SIGS = {"tier_file_open": (C.c_int, [C.c_char_p, i64, PP]),
             "tier_file_direct": (C.c_int, [P]),
             "tier_file_close": (C.c_int, [P]),
             "tier_file_write": (C.c_int, [P, P, i64, i32]),
             "tier_file_read": (C.c_int, [P, P, i64, i32])}
# multi-GPU profile exchange (kvt_ product, orc_ restatement)
MERGE_SIGS = {"pset_record_bytes": (i64, [i32, i32, i32]),
              "pset_record_pack": (C.c_int, [C.POINTER(Profiles), P]),
              "pset_merge": (C.c_int, [P, P, i32, i32, i32, i32, PP])}
# ref_insert_joint_cached: the CPU cached-greedy baseline (oracle/ref_capi.cpp), same signature
CACHED_SIGS = {"insert_joint_cached": PLACEMENT_SIGS["insert_joint"]}
# kvt_oracle_mckp (product) / ref_oracle_mckp (reference glue): bound when exported
MCKP_SIGS = {"oracle_mckp": (C.c_int, [P, P, C.POINTER(Tier), i32, C.POINTER(Space), C.POINTER(Params), f64,
                                       C.POINTER(C.c_double), P])}


class AbiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class ValidationError(AbiError):
    """Maps kvtier::ValidationError (proj/include/kvtier/core.hpp:18-20)."""


class Abi:
    """Binds one implementation of the ABI (`prefix` in kvt_/orc_/ref_)."""

    def __init__(self, path: str, prefix: str, codec: bool = True, extra: bool = False):
        if not os.path.exists(path):
            raise FileNotFoundError(f"shared library not found: {path}")
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        sigs = dict(PLACEMENT_SIGS)
        if codec:
            sigs.update(CODEC_SIGS)
        if extra:
            sigs.update(PRODUCT_EXTRA_SIGS)
        if hasattr(self.lib, prefix + "tier_moves"):
            sigs.update(TIER_SIGS)
        if hasattr(self.lib, prefix + "tier_file_open"):
            sigs.update(FILE_SIGS)
        if hasattr(self.lib, prefix + "oracle_mckp"):
            sigs.update(MCKP_SIGS)
        if hasattr(self.lib, prefix + "pset_merge"):
            sigs.update(MERGE_SIGS)
        if hasattr(self.lib, prefix + "insert_joint_cached"):
            sigs.update(CACHED_SIGS)
        for name, (res, args) in sigs.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)

    def check(self, rc):
        if rc != KVT_OK:
            msg = self.last_error().decode(errors="replace")
            if rc == KVT_EVALIDATION:
                raise ValidationError(rc, msg)
            raise AbiError(rc, msg)
        return rc


def ptr(a):
    """Address of a numpy array / torch tensor / None for a void* argument."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
