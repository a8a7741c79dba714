"""Boundary behaviour the reference's callers rely on.

* validate_hierarchy rejections (proj/src/core.cpp:86-121, pinned by
  proj/tests/test_core.cpp:66-125): every broken hierarchy is refused with
  the reference's own ValidationError message, by the oracle (CPU) and the
  CUDA library (GPU), compared live against the reference build.
* Re-entrancy (the reference runs independent stores on worker threads under
  `kvtier compare --jobs`, proj/tools/kvtier_main.cpp:206-235): two handles
  driven from two threads, interleaving insert_joint and compress, give the
  results a single thread gets.
* Handle lifetime: the tier-move streams and events belong to the handle and
  die with it (create / move / destroy many times).
"""
import ctypes as C
import threading

import numpy as np
import pytest

from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import CandidateSpace, Engine, TierSpec, UtilityParams

from cases import random_instance


def _broken_hierarchies():
    fast = dict(tier_id=0, name="fast", capacity_bytes=8_000_000_000, read_bandwidth=20e9)
    slow = dict(tier_id=1, name="slow", capacity_bytes=None, read_bandwidth=2e9)
    T = lambda **kw: TierSpec(**kw)  # noqa: E731
    return {
        # proj/tests/test_core.cpp:105-124
        "unlimited_above_finite": [T(**{**fast, "capacity_bytes": None}), T(**{**slow, "capacity_bytes": 8_000_000_000})],
        "duplicate_ids": [T(**fast), T(**{**slow, "tier_id": 0})],
        "zero_bandwidth": [T(**{**fast, "read_bandwidth": 0.0}), T(**slow)],
        "empty": [],
        # the remaining throws of core.cpp:102-110
        "negative_capacity": [T(**{**fast, "capacity_bytes": -1}), T(**slow)],
        "nan_bandwidth": [T(**fast), T(**{**slow, "read_bandwidth": float("nan")})],
        "inf_bandwidth": [T(**{**fast, "read_bandwidth": float("inf")}), T(**slow)],
        "negative_latency": [T(**fast), T(**{**slow, "fixed_access_latency": -1e-3})],
        "inf_latency": [T(**{**fast, "fixed_access_latency": float("inf")}), T(**slow)],
        # accepted: unsorted input (test_core.cpp:66-74), a lone unlimited tier (:92-98),
        # bandwidth growing down the stack (a warning only, :127-133)
        "ok_unsorted": [T(**slow), T(**fast)],
        "ok_single_unlimited": [T(tier_id=0, name="remote", capacity_bytes=None, read_bandwidth=1e9)],
        "ok_bandwidth_grows": [T(**fast), T(**{**slow, "read_bandwidth": 40e9})],
    }


def _outcome(eng, tiers):
    """What the library does with `tiers`: 'ok' or (status class, message)."""
    arrays, _, space, params = random_instance(3, n_ctx=5, n_methods=2, n_tiers=2)
    ps = eng.pset(arrays)
    try:
        eng.score_candidates(ps, tiers, space, params)
        eng.store(tiers, arrays.n, space)
    except A.ValidationError as e:
        return ("ValidationError", str(e))
    return "ok"


def _check_hierarchy_parity(eng, ref_abi):
    er = Engine(ref_abi)
    for name, tiers in _broken_hierarchies().items():
        got, want = _outcome(eng, tiers), _outcome(er, tiers)
        assert got == want, f"{name}: {got} vs reference {want}"
        assert (want == "ok") == name.startswith("ok_"), f"{name}: reference outcome {want}"


def test_oracle_validate_hierarchy_matches_reference(oracle_abi, ref_abi):
    _check_hierarchy_parity(Engine(oracle_abi), ref_abi)


@pytest.mark.gpu
def test_gpu_validate_hierarchy_matches_reference(gpu_abi, ref_abi):
    _check_hierarchy_parity(Engine(gpu_abi), ref_abi)


def _placement_run(eng, seed):
    arrays, tiers, space, params = random_instance(seed, n_ctx=60, n_methods=3, n_tiers=3)
    ps = eng.pset(arrays)
    st = eng.store(tiers, arrays.n, space)
    acts = st.insert_joint(ps, space, params, np.arange(arrays.n))
    return acts, st.snapshot(), st.placement_utility(ps, space, params)


def _codec_run(eng, seed):
    import torch
    s = A.KvShape(2, 2, 512, 128)
    cfg = A.CodecCfg()
    eng.abi.check(eng.abi.codec_plan(b"keydiff-q4", 0.2, C.byref(s), C.byref(cfg)))
    m = A.BlobMap()
    eng.abi.check(eng.abi.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    n = 2 * 2 * 512 * 128
    k = torch.empty(n, dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    eng.abi.check(eng.abi.kv_generate(eng.h, C.byref(s), 11, seed, A.ptr(k), A.ptr(v)))
    ws = torch.empty(eng.abi.compress_workspace_bytes(C.byref(s), C.byref(cfg)), dtype=torch.uint8, device="cuda")
    blob = torch.zeros(m.total_bytes, dtype=torch.uint8, device="cuda")
    eng.abi.check(eng.abi.compress(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws), A.ptr(blob)))
    eng.abi.check(eng.abi.sync(eng.h))
    return blob.cpu().numpy()


@pytest.mark.gpu
def test_gpu_two_handles_two_threads(gpu_abi):
    """Independent stores on worker threads (compare --jobs): each thread
    owns a handle on its own stream and interleaves insert_joint with
    compress; every result equals the single-threaded one."""
    import torch
    seeds = [21, 22]
    want = {}
    for sd in seeds:
        e = Engine(gpu_abi)
        want[sd] = (_placement_run(e, sd), _codec_run(e, sd))
        e.close()
    got, errs = {}, []

    def worker(sd):
        try:
            st = torch.cuda.Stream()
            e = Engine(gpu_abi, stream=st.cuda_stream)
            res = []
            for _ in range(3):
                res.append((_placement_run(e, sd), _codec_run(e, sd)))
            got[sd] = res
            e.close()
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=worker, args=(sd,)) for sd in seeds]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for sd in seeds:
        (wa, ws, wu), wb = want[sd]
        for (ga, gs, gu), gb in got[sd]:
            assert np.array_equal(ga, wa) and np.array_equal(gs, ws) and gu == wu
            assert np.array_equal(gb, wb)


@pytest.mark.gpu
def test_gpu_handle_owns_move_streams(gpu_abi):
    """kvt_destroy releases the handle's copy streams and events: 64
    create / move / destroy cycles, each round trip exact."""
    import torch
    from paper_2512_14946_b200.tiers import HostArena
    src = torch.arange(1 << 20, dtype=torch.int32, device="cuda").view(torch.uint8)
    for i in range(64):
        e = Engine(gpu_abi)
        arena = HostArena(e.abi, src.numel())
        mv = (A.Move * 1)(A.Move(src.data_ptr(), arena.base, src.numel(), A.KVT_MOVE_D2H, 0))
        e.abi.check(e.abi.tier_moves(e.h, mv, 1))
        e.abi.check(e.abi.sync(e.h))
        host = np.ctypeslib.as_array((C.c_uint8 * src.numel()).from_address(arena.base))
        assert np.array_equal(host, src.cpu().numpy())
        arena.close()
        e.close()
