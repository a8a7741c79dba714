"""Per-kernel probe of the hot path on one full Llama-3.1-8B KV chunk
(32 L x 8 H x 8192 T x 128 D, 1 GiB bf16) and the c2 placement pass.

Runs every codec phase as its own C-ABI call so each kernel is separately
visible to ncu, and prints one JSON line per phase with CUDA-event times and
the algorithmic bytes of DESIGN.md §Roofline. Used for the launch lists and
`ncu --set full` captures committed under profiles/; numbers printed while
running under ncu are not bench values.

  python profiles/codec_probe.py [--reps 3] [--methods knorm-q4:0.2,...]
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

import paper_2512_14946_b200 as pkg  # noqa: E402
from paper_2512_14946_b200 import _abi as A  # noqa: E402
from paper_2512_14946_b200.kvtier import Engine  # noqa: E402

DEFAULT = "knorm-q4:0.2,keydiff-q4:0.2,snapkv-q4:0.2,knorm-q8:0.4,knorm:0.4,knorm-q2:0.1"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--methods", default=DEFAULT)
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--L", type=int, default=32)
    args = ap.parse_args()

    eng = Engine(pkg.product())
    ab = eng.abi
    s = A.KvShape(args.L, 8, args.T, 128)
    n = s.L * s.H * s.T * s.D
    k = torch.empty(n, dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    ab.check(ab.kv_generate(eng.h, C.byref(s), 1, 0, A.ptr(k), A.ptr(v)))
    peak = 6543.1
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = json.load(f)["hbm_gbs"]
    except Exception:
        pass
    for spec in args.methods.split(","):
        meth, ratio = spec.split(":")
        cfg = A.CodecCfg()
        ab.check(ab.codec_plan(meth.encode(), float(ratio), C.byref(s), C.byref(cfg)))
        m = A.BlobMap()
        ab.check(ab.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
        S = s.L * s.H
        sc = torch.empty(S * s.T, dtype=torch.float32, device="cuda")
        idx = torch.zeros(S * cfg.keep, dtype=torch.int32, device="cuda")
        blob = torch.empty(m.total_bytes, dtype=torch.uint8, device="cuda")
        ws = torch.zeros(ab.compress_workspace_bytes(C.byref(s), C.byref(cfg)), dtype=torch.uint8, device="cuda")
        kk = cfg.keep
        alg = {
            "scores": S * s.T * 256 + S * s.T * 4,
            "topk": S * s.T * 4 + S * kk * 4,
            "pack": 2 * S * kk * 256 + m.total_bytes,
            "compress": S * s.T * 256 + S * kk * 256 + m.total_bytes,
            "unpack": m.total_bytes + 2 * S * kk * 256,
        }
        ku = torch.empty(S * kk * 128, dtype=torch.int16, device="cuda")
        vu = torch.empty_like(ku)
        acc = {p: 0.0 for p in alg}
        for r in range(args.reps + 1):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            ev[0].record()
            ab.check(ab.token_scores(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(sc)))
            ev[1].record()
            ab.check(ab.topk(eng.h, C.byref(s), C.byref(cfg), A.ptr(sc), A.ptr(idx)))
            ev[2].record()
            ab.check(ab.pack(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), A.ptr(idx), A.ptr(blob)))
            ev[3].record()
            ab.check(ab.compress(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws), A.ptr(blob)))
            ev[4].record()
            if cfg.bits < 16:
                ab.check(ab.unpack(eng.h, C.byref(s), C.byref(cfg), A.ptr(blob), A.ptr(ku), A.ptr(vu)))
            ev[5].record()
            torch.cuda.synchronize()
            if r == 0:
                continue  # warm-up
            for i, p in enumerate(("scores", "topk", "pack", "compress", "unpack")):
                acc[p] += ev[i].elapsed_time(ev[i + 1]) / max(1, args.reps)
        out = {"method": meth, "ratio": float(ratio), "bits": cfg.bits, "keep": kk, "T": s.T, "L": s.L}
        for p in alg:
            gbs = alg[p] / (acc[p] / 1e3) / 1e9 if acc[p] > 0 else 0.0
            out[p] = {"ms": round(acc[p], 4), "alg_bytes": alg[p], "GBps": round(gbs, 1), "frac": round(gbs / peak, 4)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
