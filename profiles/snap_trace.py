"""Timeline probe of k_snapkv_tc: builds nothing, loads the trace build
(`make -C paper_2512_14946_b200/csrc trace` -> build_trace/libkvt_trace.so,
compiled with -DKVT_SNAP_TRACE) and prints, for the first cluster's rank-0
CTA, when each tile's bf16 stage landed / its MMA was issued (producer
thread 0) and when consumer warp 0 got / finished its epilogue block, then
the slice tail's rounds. Times in microseconds from kernel start. Probe
only: the product library has no trace points.

  python profiles/snap_trace.py [--T 8192] [--L 32] [--sms 0]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_14946_b200 import _abi as A  # noqa: E402
from paper_2512_14946_b200.kvtier import Engine  # noqa: E402

TAIL = ["tiles_done", "round0", "round1", "weights", "vote", "halo", "end"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--slices", type=int, default=4, help="slices of the first cluster to print")
    args = ap.parse_args()
    lib = os.path.join(ROOT, "paper_2512_14946_b200", "csrc", "build_trace", "libkvt_trace.so")
    ab = A.Abi(lib, "kvt_", codec=True, extra=True)
    eng = Engine(ab)
    s = A.KvShape(args.L, 8, args.T, 128)
    n = s.L * s.H * s.T * s.D
    k = torch.empty(n, dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    ab.check(ab.kv_generate(eng.h, C.byref(s), 1, 0, A.ptr(k), A.ptr(v)))
    cfg = A.CodecCfg()
    ab.check(ab.codec_plan(b"snapkv-q4", 0.2, C.byref(s), C.byref(cfg)))
    sc = torch.empty(s.L * s.H * s.T, dtype=torch.float32, device="cuda")
    for _ in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        ab.check(ab.token_scores(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(sc)))
        ev[1].record()
        torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    buf = (C.c_ulonglong * 4096)()
    fn = ab.lib.kvt_debug_snap_trace
    fn.argtypes = [C.c_void_p, C.c_int]
    assert fn(C.cast(buf, C.c_void_p), 4096) == 0
    t0 = buf[4000]
    rel = lambda x: round((x - t0) / 1e3, 2) if x >= t0 and x else None  # noqa: E731
    out = {"kernel_ms": round(ms, 4), "prod_end": rel(buf[4001]), "cons_end": rel(buf[4002]), "slices": []}
    for it in range(64):
        b = it * 64
        if not buf[b + 38] or buf[b + 38] < t0:
            break
        sl = {
            "it": it,
            "stage_full": [rel(buf[b + 2 * j]) for j in range(8)],
            "mma_issued": [rel(buf[b + 2 * j + 1]) for j in range(8)],
            "cons_get": [rel(buf[b + 16 + 2 * j]) for j in range(8)],
            "cons_done": [rel(buf[b + 16 + 2 * j + 1]) for j in range(8)],
        }
        for i, name in enumerate(TAIL):
            sl[name] = rel(buf[b + 32 + i])
        out["slices"].append(sl)
    print(json.dumps({k_: v_ for k_, v_ in out.items() if k_ != "slices"}))
    for sl in out["slices"][: args.slices]:
        print(json.dumps(sl))
    # cluster 0's CTAs: when each finished its tiles (skew the first round waits for)
    skew = []
    for it in range(min(16, len(out["slices"]))):
        ts = [buf[2048 + it * 16 + r] for r in range(16)]
        ts = [t for t in ts if t >= t0 and t]
        if ts:
            skew.append(round((max(ts) - min(ts)) / 1e3, 2))
    print(json.dumps({"tiles_done_skew_us": skew}))
    # per-slice durations
    ends = [sl["end"] for sl in out["slices"]]
    print(json.dumps({"n_slices": len(ends), "slice_period_us": [round(b - a, 2) for a, b in zip(ends, ends[1:])]}))


if __name__ == "__main__":
    main()
