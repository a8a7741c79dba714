"""Bench: KV GB/s compressed + scored + placed (BASELINE.json metric).

One step = one pass of the hot path over a batch of contexts with inputs
resident in HBM: K1 candidate scoring + K3 greedy placement of every context
(insert_joint in arrival order into an empty 3-tier store), then the codec
(token scores -> per-head top-k -> gather + quantise + pack) of every
context's KV chunk at the configuration it was placed at. value = original
KV bytes of the batch / device time of the step, summed over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
  python bench.py --impl reference   # CPU reference arm (oracle/_ref + codec port)

N > 1: one process per GPU (torchrun; `--gpus N` without torchrun re-launches
itself under torch.distributed.run). Each rank owns n_ctx contexts (weak
scaling). The placement is global: every step, each rank's profile record is
all-gathered over NCCL (inside the timed region) and merged into the global
profile set on the device (kvt_pset_merge); every rank runs the identical
deterministic greedy over all contexts, then compresses only its own.

Lines: `value` (inputs resident in HBM), `e2e` (profile rows H2D from pinned
host memory + action list and placement D2H every step, through the C ABI),
`e2e_tiered` (e2e plus the tier moves the placement implies: every context
placed below the GPU tier leaves HBM over PCIe), `roofline`, `tier_move`
(PCIe and SSD rates, verified), `cpu_baseline`.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- helpers

def algorithmic_bytes(L, H, T, cfg, m):
    """Per-launch algorithmic HBM bytes of each codec phase."""
    S, D, k = L * H, 128, cfg.keep
    kv_rows = S * T * D * 2
    return {
        "scores": kv_rows + S * T * 4,                          # read K once, write f32 scores
        "topk": S * T * 4 + S * k * 4,                          # read scores, write indices
        "pack": 2 * S * k * D * 2 + (m.total_bytes),            # read kept K,V rows, write blob
    }


SCORER_KERNEL = {0: "k_knorm", 1: "k_keydiff_cluster", 2: "k_snapkv_tc"}


def traffic_table():
    """ncu-measured DRAM bytes per launch (dram__bytes_read.sum +
    dram__bytes_write.sum, one --set full capture per kernel on one full
    Llama-3.1-8B chunk), committed under profiles/; None when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def kernel_roofline(eng, stream, codec, pool, store, arrays, space, L, H, D, bpt, lo, hi):
    """One instrumented pass over this rank's contexts, every codec phase
    its own C-ABI call bracketed by CUDA events on the launching stream:
    time and algorithmic bytes per kernel (scores per scorer, top-k, pack per
    bit width), the dominant kernel's roofline, and per-phase shares."""
    import torch

    from paper_2512_14946_b200 import _abi as A

    snap = store.snapshot()
    names = space.method_names
    recs = []
    # hold the stream ~50 ms so the host enqueues the pass ahead of the GPU:
    # a host stall between an event and its launch must not count as kernel time
    with torch.cuda.stream(stream):
        torch.cuda._sleep(100_000_000)
    n_identity = 0
    for c in range(lo, hi):
        if snap["tier_index"][c] < 0:
            continue
        T = int(arrays.orig[c] // bpt)
        cfgc, m, wsb = codec.plan(names[snap["method"][c]], float(snap["ratio"][c]), T)
        if m.identity:  # the compressed chunk is the source KV: no kernel, no bytes
            n_identity += 1
            continue
        s = A.KvShape(L, H, T, D)
        k, v = pool.chunk(c)
        sc = codec.ws  # scores at offset 0
        idx = codec.ws.data_ptr() + wsb - ((4 * L * H * cfgc.keep + 255) // 256) * 256
        ab = algorithmic_bytes(L, H, T, cfgc, m)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        full = cfgc.keep == T  # every token kept: compress skips scoring and selection
        if full:  # indices 0..T-1 (what kvt_compress writes), outside the timed phases
            eng.abi.check(eng.abi.topk(eng.h, C.byref(s), C.byref(cfgc), A.ptr(sc), idx))
        evs[0].record(stream)
        if not full:
            eng.abi.check(eng.abi.token_scores(eng.h, C.byref(s), C.byref(cfgc), A.ptr(k), None, A.ptr(sc)))
        evs[1].record(stream)
        if not full:
            eng.abi.check(eng.abi.topk(eng.h, C.byref(s), C.byref(cfgc), A.ptr(sc), idx))
        evs[2].record(stream)
        eng.abi.check(eng.abi.pack(eng.h, C.byref(s), C.byref(cfgc), A.ptr(k), A.ptr(v), idx, A.ptr(codec.out[0])))
        evs[3].record(stream)
        keys = [None if full else SCORER_KERNEL[cfgc.scorer], None if full else "k_topk",
                "k_gather16" if cfgc.bits == 16 else f"k_pack_kv<{cfgc.bits}>"]
        recs.append((evs, keys, [ab["scores"], ab["topk"], ab["pack"]]))
    torch.cuda.synchronize()
    per = {}
    phase = {"scores": 0.0, "topk": 0.0, "pack": 0.0}
    step_bytes = sum(ab for evs, keys, abs_ in recs for key, ab in zip(keys, abs_) if key is not None)
    for evs, keys, abs_ in recs:
        for i, (key, ph) in enumerate(zip(keys, ("scores", "topk", "pack"))):
            if key is None:
                continue
            dt = evs[i].elapsed_time(evs[i + 1])
            e = per.setdefault(key, [0.0, 0, 0])
            e[0] += dt
            e[1] += abs_[i]
            e[2] += 1
            phase[ph] += dt
    tot = sum(phase.values())
    dom = max(per, key=lambda k_: per[k_][0])
    t_ms, alg, n = per[dom]
    pk, how = peaks()
    achieved = alg / (t_ms / 1e3) / 1e9
    traffic = traffic_table().get(dom)
    line = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4),
            "traffic": traffic, "traffic_note": "ncu dram read+write bytes per launch (profiles/traffic.json)",
            "alg_bytes_per_launch": int(alg // n), "avg_launch_ms": round(t_ms / n, 4), "launches": n,
            "peak_source": how, "time_share": round(t_ms / tot, 4),
            "phase_share": {ph: round(v / tot, 4) for ph, v in phase.items()},
            "kernels": {k_: {"ms": round(v[0], 2), "n": v[2], "GBps": round(v[1] / (v[0] / 1e3) / 1e9, 1),
                             "frac": round(v[1] / (v[0] / 1e3) / 1e9 / pk["hbm_gbs"], 4)}
                        for k_, v in sorted(per.items(), key=lambda kv: -kv[1][0])}}
    if dom in ISSUE_BOUND:  # HBM fraction is reported, but it is not what bounds this kernel
        line["bound_note"] = ISSUE_BOUND[dom]
    line["identity_contexts"] = n_identity
    line["alg_bytes_per_step_rank"] = int(step_bytes)
    line["unpack"] = unpack_rate(eng, stream, codec, pool, snap, arrays, names, L, H, D, bpt, lo, hi)
    ge = os.environ.get("KVT_SNAP_SMS")
    if dom == "k_snapkv_tc" and ge:  # runs on a share of the SMs by design (the step's other streams get the rest)
        sms = min(int(ge), torch.cuda.get_device_properties(0).multi_processor_count)
        line["sms"] = sms
        line["frac_per_sm"] = round(line["frac"] * torch.cuda.get_device_properties(0).multi_processor_count / sms, 4)
    return line


def unpack_rate(eng, stream, codec, pool, snap, arrays, names, L, H, D, bpt, lo, hi, per_bits=3):
    """k_unpack (unpack + dequantise, the decompression half of north-star
    item 1): a few placed quantised contexts per bit width, compressed then
    unpacked into bf16 [L][H][keep][D], CUDA events on the launching stream.
    Algorithmic bytes per launch = blob + 2 x 2 B x L H keep D."""
    import torch

    from paper_2512_14946_b200 import _abi as A
    pk, _ = peaks()
    seen, out = {}, {}
    for c in range(lo, hi):
        if snap["tier_index"][c] < 0:
            continue
        T = int(arrays.orig[c] // bpt)
        meth, ratio = names[snap["method"][c]], float(snap["ratio"][c])
        cfgc, m, _ = codec.plan(meth, ratio, T)
        if m.identity or cfgc.bits == 16 or seen.get(cfgc.bits, 0) >= per_bits:
            continue
        seen[cfgc.bits] = seen.get(cfgc.bits, 0) + 1
        k, v = pool.chunk(c)
        s_ = A.KvShape(L, H, T, D)
        blob = torch.empty(m.total_bytes, dtype=torch.uint8, device="cuda")
        eng.abi.check(eng.abi.compress(eng.h, C.byref(s_), C.byref(cfgc), A.ptr(k), A.ptr(v), None,
                                       A.ptr(codec.ws), A.ptr(blob)))
        n = L * H * cfgc.keep * D
        ko = torch.empty(n, dtype=torch.int16, device="cuda")
        vo = torch.empty_like(ko)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.abi.check(eng.abi.unpack(eng.h, C.byref(s_), C.byref(cfgc), A.ptr(blob), A.ptr(ko), A.ptr(vo)))  # warm
        e0.record(stream)
        eng.abi.check(eng.abi.unpack(eng.h, C.byref(s_), C.byref(cfgc), A.ptr(blob), A.ptr(ko), A.ptr(vo)))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        alg = m.total_bytes + 2 * 2 * n
        r = out.setdefault(f"q{cfgc.bits}", {"ms": 0.0, "bytes": 0, "n": 0})
        r["ms"] += ms
        r["bytes"] += alg
        r["n"] += 1
    for r in out.values():
        gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9
        r.update(GBps=round(gbs, 1), frac=round(gbs / pk["hbm_gbs"], 4), avg_launch_ms=round(r["ms"] / r["n"], 4),
                 ms=round(r["ms"], 3))
    return {"kernel": "k_unpack", "by_bits": out,
            "note": "alg bytes = blob + 4 B x L H keep D (bf16 K and V out); placed contexts of this batch"}


# kernels whose limit is instruction issue, not HBM (ncu captures in profiles/)
ISSUE_BOUND = {
    "k_snapkv_tc": "issue-bound: the exp epilogue (FMA + ALU pipes, 1 exp per logit, 268 M logits per chunk) "
                   "and the per-slice cluster tail; DRAM 548 MB/launch = 1.00x algorithmic; ncu issue active 66 %, "
                   "173 M warp-instructions per launch (profiles/r3d_ncu_snapkv_raw.csv, "
                   "r3d_ncu_snapkv_source_summary.txt, DESIGN.md §5)",
    "k_keydiff_cluster": "issue/latency-bound: K is read from HBM once (574 MB/launch with the L2 hints); "
                         "ncu issue active 60 %, 97 M warp-instructions (profiles/r2m_ncu_keydiff_raw.csv)",
}


def tier_move_rates(eng, stream, codec, pool, snap, arrays, space, L, H, D, bpt, lo, hi, n_ctx=4, reps=3,
                    ssd_bytes=4 << 30):
    """SURVEY §8 f1 evidence. PCIe: pinned cudaMemcpyAsync GB/s of
    kvt_tier_moves moving the compressed bytes of contexts the greedy placed
    below the GPU tier to the pinned CPU-tier arena (D2H) and back into fresh
    device buffers (H2D), CUDA events on the handle stream; both directions
    are verified byte for byte before timing. SSD: up to `ssd_bytes` of
    SSD-tier contexts staged through pinned DRAM and written to a file with
    kvt_tier_file_write (O_DIRECT, threads), read back and verified."""
    import tempfile

    import torch

    from paper_2512_14946_b200 import _abi as A
    from paper_2512_14946_b200.tiers import HostArena, SsdTier, TierExecutor, context_sources, host_moves_bytes

    names = space.method_names

    def compressed(c):
        T = int(arrays.orig[c] // bpt)
        cfgc, m, _ = codec.plan(names[snap["method"][c]], float(snap["ratio"][c]), T)
        s_ = A.KvShape(L, H, T, D)
        k, v = pool.chunk(c)
        b = torch.empty(max(1, m.total_bytes), dtype=torch.uint8, device="cuda")
        eng.abi.check(eng.abi.compress(eng.h, C.byref(s_), C.byref(cfgc), A.ptr(k), A.ptr(v), None,
                                       A.ptr(codec.ws), A.ptr(b)))
        return [(p_, n_) for p_, n_ in context_sources(b.data_ptr(), m, k.data_ptr(), v.data_ptr(), k.numel() * 2)], b

    # ---- PCIe leg: CPU-tier (and SSD-tier) contexts, device <-> pinned host
    srcs, keep = [], []
    for c in range(lo, hi):
        if snap["tier_index"][c] > 0 and len(keep) < n_ctx:
            r_, b = compressed(c)
            srcs += r_
            keep.append(b)
    if not srcs:
        return None
    total = sum(n_ for _, n_ in srcs)
    arena = HostArena(eng.abi, total + (1 << 20))
    ex = TierExecutor(eng, arena)
    down = ex.moves_for([(i, 1, p_, n_) for i, (p_, n_) in enumerate(srcs)])
    fresh = [torch.empty(n_, dtype=torch.uint8, device="cuda") for _, n_ in srcs]
    up = [A.Move(mv.dst, t.data_ptr(), mv.bytes, A.KVT_MOVE_H2D, 0) for mv, t in zip(down, fresh)]
    ex.run(down)
    eng.abi.check(eng.abi.sync(eng.h))
    ok = True
    for (p_, n_), mv in zip(srcs, down):  # host copy == device bytes, right after the D2H
        ok &= bool(np.array_equal(arena.view(mv.dst, mv.bytes), _device_bytes(p_, n_)))
    ex.run(up)
    eng.abi.check(eng.abi.sync(eng.h))
    for (p_, n_), t in zip(srcs, fresh):  # H2D into fresh buffers == the original device bytes
        ok &= bool(np.array_equal(t.cpu().numpy(), _device_bytes(p_, n_)))
    rates = {}
    for name, mv in (("d2h", down), ("h2d", up)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            ex.run(mv)
        e1.record(stream)
        torch.cuda.synchronize()
        rates[name] = host_moves_bytes(mv) * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    out = {"d2h_gbs": round(rates["d2h"], 1), "h2d_gbs": round(rates["h2d"], 1), "bytes": int(total),
           "contexts": len(keep), "verified": bool(ok),
           "note": "kvt_tier_moves: compressed bytes of below-GPU-tier contexts (source K/V for identity "
                   "configurations), device -> pinned host, then host -> fresh device buffers; 8 MiB pieces "
                   "over 2 copy streams per direction; each direction verified byte for byte before timing"}
    arena.close()

    # ---- SSD leg: SSD-tier contexts, staged through pinned DRAM, into a file
    ssd_src = []
    for c in range(lo, hi):
        if snap["tier_index"][c] == 2 and sum(n_ for _, n_ in ssd_src) < ssd_bytes:
            r_, b = compressed(c)
            ssd_src += r_
            keep.append(b)
    if ssd_src:
        nb = sum(n_ for _, n_ in ssd_src)
        d = os.environ.get("KVT_SSD_DIR") or tempfile.gettempdir()
        st_ = os.statvfs(d)
        if st_.f_bavail * st_.f_frsize < 2 * nb + (1 << 30):
            out["ssd"] = {"skipped": f"not enough free space in {d}"}
            return out
        stage = HostArena(eng.abi, nb + 64 * 4096)
        back = HostArena(eng.abi, nb + 64 * 4096)
        ex2 = TierExecutor(eng, stage)
        mv = ex2.moves_for([(i, 2, p_, n_) for i, (p_, n_) in enumerate(ssd_src)])
        ex2.run(mv)
        eng.abi.check(eng.abi.sync(eng.h))
        ssd = SsdTier(eng.abi, os.path.join(d, f"kvt_ssd_tier_{os.getpid()}.bin"), nb + 64 * 4096, threads=8)
        offs = [ssd.alloc(m_.bytes) for m_ in mv]
        t0 = time.perf_counter()
        ssd.write([(m_.dst, m_.bytes, o) for m_, o in zip(mv, offs)])
        t_w = time.perf_counter() - t0
        dst = [back.slot(i, m_.bytes) for i, m_ in enumerate(mv)]
        t0 = time.perf_counter()
        ssd.read([(a, m_.bytes, o) for a, m_, o in zip(dst, mv, offs)])
        t_r = time.perf_counter() - t0
        ok2 = all(np.array_equal(back.view(a, m_.bytes), _device_bytes(p_, n_))
                  for a, m_, (p_, n_) in zip(dst, mv, ssd_src))
        out["ssd"] = {"write_gbs": round(nb / t_w / 1e9, 2), "read_gbs": round(nb / t_r / 1e9, 2), "bytes": int(nb),
                      "o_direct": ssd.direct, "dir": d, "verified": bool(ok2), "threads": 8,
                      "note": "SSD-tier contexts: HBM -> pinned DRAM (kvt_tier_moves) -> file (kvt_tier_file_write, "
                              "fdatasync), read back (kvt_tier_file_read) and compared with the device bytes; "
                              "the read may be served from the page cache when O_DIRECT is unavailable"}
        ssd.close()
        stage.close()
        back.close()
    return out


def _device_bytes(ptr, n):
    """Copy n device bytes at `ptr` to a host numpy array (cudaMemcpy via torch)."""
    return _alias(ptr, n).cpu().numpy()


def _alias(ptr, n):
    """A torch uint8 CUDA tensor viewing n bytes at device address `ptr`."""
    import torch

    class _Cai:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_Cai(), device="cuda")


# snapkv's SM budget in the split schedule, per workload: A/B on one B200
# (alternating runs, same box): c2 48 SMs 3,507 / 56 3,475 / 64 3,453 GB/s;
# c5 (varied lengths, up to 16-CTA clusters) 48 3,278 / 64 3,323 GB/s;
# r2z, after the pack cuts: c3 48 / 56 / 64 3,446 / 3,507 / 3,477; c4 48 /
# 64 / 80 3,689 / 3,743 / 3,687 (profiles/r2z_c34_sms_sweep.txt).
SNAP_SMS = {"c3": 56, "c4": 64, "c5": 64}


def north_star_pass(args):
    """BASELINE configs[4] beside the headline config: the full compress +
    score + place pass over 13,889 varied-length contexts x 72 candidates =
    1,000,008 chunk-configs (the north-star target), one warm-up and
    `--n1-steps` timed steps in a child process on the same GPU. Its
    placement is the reference's own, bit for bit
    (tests/test_large_placement.py, fixture from the reference greedy)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--config", "c5", "--steps", str(args.n1_steps), "--warmup", "1",
           "--no-cpu-baseline", "--tiered-steps", "0", "--no-n1", "--snap-sms", str(SNAP_SMS.get("c5", 48)),
           "--streams", str(args.streams), "--lanes", args.lanes, "--group-slices", str(args.group_slices)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, not fatal for the headline line
        return {"error": f"{type(e).__name__}: {e}"[:300]}
    roof = d.get("roofline") or {}
    return {"workload": d["config"]["workload"], "candidates": 13889 * 72, "value": d["value"], "unit": "GB/s",
            "ms_per_step": d["ms_per_step"], "steps": d["steps"], "e2e": d["e2e"],
            "actions_per_step": d["details"]["actions_per_step"], "step_hbm_frac": roof.get("step_hbm_frac"),
            "dominant_kernel": roof.get("kernel"), "dominant_frac": roof.get("frac"),
            "gpu_launches": d.get("gpu_launches"), "clocks": d.get("clocks"),
            "parity": "placement bit-exact to the reference greedy on this instance (tests/test_large_placement.py "
                      "c5 fixture); codec kernels bit-exact to the codec oracle (tests/test_gpu_codec.py)"}


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def config_dict(args, W, n_total, world):
    """The workload description, identical in both arms (same_config)."""
    cfg, space = W["cfg"], W["space"]
    return {"workload": f"{args.config}: {cfg['model']} KV, {W['arrays'].n} contexts/GPU x {cfg['tokens']} tokens, "
                        f"{len(space.methods)} methods x {len(space.ratios)} ratios x 3 tiers",
            "contexts_total": int(n_total), "contexts_per_gpu": int(W["arrays"].n), "methods": space.method_names,
            "tiers": "gpu {:.0%} of bytes @8e12 B/s, cpu 30% @5e10, ssd unlimited @6e9 + 1e-4 s".format(
                cfg["gpu_frac"]),
            "seed": "7 + rank", "n_gpus": world}


def nccl_summary(path_glob):
    """What NCCL_DEBUG=INFO logged on this rank: communicator size, NVLS."""
    import glob
    out = {"ranks": None, "nvls": False, "lines": 0}
    for fn in glob.glob(path_glob):
        try:
            txt = open(fn, errors="replace").read()
        except OSError:
            continue
        out["lines"] += txt.count("\n")
        for ln in txt.splitlines():
            if "Init COMPLETE" in ln and "nranks" in ln:
                try:
                    out["ranks"] = int(ln.split("nranks")[1].split()[0])
                except Exception:
                    pass
            if "NVLS" in ln and ("enabled" in ln.lower() or "nvls multicast support is available" in ln.lower()):
                out["nvls"] = True
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2512_14946_b200 as pkg
    from paper_2512_14946_b200 import _abi as A
    from paper_2512_14946_b200 import distributed, workload
    from paper_2512_14946_b200.kvtier import Engine
    from paper_2512_14946_b200.pipeline import Codec, KVPool, place, split_plan
    from paper_2512_14946_b200.tiers import StagingRing, context_sources

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}; measuring {world} ranks", file=sys.stderr)
    if args.ranks_share_gpu:  # test mode: every rank on cuda:0, the exchange over gloo on host buffers
        local = 0
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench: rank {rank} needs cuda:{local}, {torch.cuda.device_count()} device(s) visible")
    torch.cuda.set_device(local)
    nccl_log = None
    if world > 1 and args.ranks_share_gpu:
        dist.init_process_group("gloo")
    elif world > 1:
        nccl_log = f"/tmp/kvt_bench_nccl.{os.getpid()}.log"
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log)  # keep stdout to the one JSON line
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    W = workload.build(args.config, n_ctx=args.n_ctx, seed=7 + rank)
    cfg, shape, space, mine, params = W["cfg"], W["shape"], W["space"], W["arrays"], W["params"]
    L, H, D = shape["L"], shape["H"], shape["D"]
    bpt = W["bytes_per_token"]
    n_local = mine.n

    stream = torch.cuda.Stream()
    eng = Engine(pkg.product(), device=local, stream=stream.cuda_stream)
    # this rank's profile record: pinned on the host (the e2e leg copies it in
    # every step) and resident on the device (the value leg); all-gathered over
    # NCCL and merged on the device into the global profile set
    with torch.cuda.stream(stream):
        rp = (distributed.RankPlacement(eng, mine, device="cpu", merge_on=f"cuda:{local}") if args.ranks_share_gpu
              else distributed.RankPlacement(eng, mine, device=f"cuda:{local}", pin=True))
    tot = torch.tensor([int(mine.orig.sum())], dtype=torch.int64, device="cpu" if args.ranks_share_gpu else "cuda")
    if world > 1:
        dist.all_reduce(tot)
    total_bytes = int(tot.item())  # every rank's contexts
    tiers = workload.three_tiers(total_bytes, cfg["gpu_frac"], 0.30)
    n_total = world * n_local
    my_lo, my_hi = distributed.shard(n_total, world, rank)
    assert my_hi - my_lo == n_local

    max_T = int(mine.orig.max() // bpt)
    pool = KVPool(eng, L, H, max_T, D, n_chunks=args.pool)
    # stream priorities (lower = higher priority): "snap" favours the snapkv
    # stream's launches, "mem" the memory streams'; default none
    prio = {"none": [0] * args.streams, "snap": [-1] + [0] * (args.streams - 1),
            "mem": [0] + [-1] * (args.streams - 1)}[args.lane_priority]
    lane_streams = [torch.cuda.Stream(priority=p_) for p_ in prio]
    lanes = [Engine(pkg.product(), device=local, stream=ls.cuda_stream) for ls in lane_streams]
    codec = Codec(lanes, L, H, D)
    codec.reserve(max_T, n_out=2)
    codec.attach_streams(lane_streams, ring=args.ring)
    with torch.cuda.stream(stream):
        ps_static = rp.exchange()  # the global set once (value leg at N = 1 reuses it)
    store = eng.store(tiers, n_total, space)
    order = np.arange(n_total, dtype=np.int32)
    names = space.method_names
    kv_bytes = L * H * max_T * D * 2
    staging = None  # pinned landing slots of the tiered leg

    def fork():  # codec lanes start after everything queued on the main stream
        for ls in lane_streams:
            ls.wait_stream(stream)

    def join():  # the main stream (timing events) waits for every lane
        for ls in lane_streams:
            stream.wait_stream(ls)

    def placed(upload, exchange):
        """One batch's placement on the main stream: [H2D of this rank's
        record] -> [NCCL all-gather + device merge] -> greedy -> action list
        and placement D2H (the host needs them to launch its compressions)."""
        with torch.cuda.stream(stream):
            if upload:
                rp.upload()
            ps = rp.exchange() if exchange else ps_static
        acts = place(store, ps, space, params, order)
        return acts, store.snapshot()

    def launch_compress(snap_full, tiered):
        in_b = out_b = moved = 0
        fork()
        cs = [c for c in range(my_lo, my_hi) if snap_full["tier_index"][c] >= 0]
        ms = [names[snap_full["method"][c]] for c in cs]
        rs = [float(snap_full["ratio"][c]) for c in cs]
        Ts = [int(mine.orig[c - my_lo] // bpt) for c in cs]
        plan = (split_plan(ms, rs, Ts, len(lanes), args.snap_sms) if args.lanes == "split"
                else [(None, None)] * len(cs))
        for c, m, r, T, (sl, pl) in zip(cs, ms, rs, Ts, plan):
            k, v = pool.chunk(c)
            if args.lanes == "split":
                out_b += (codec.compress(m, r, k, v, T, c, pl, group=args.group_slices) if sl is None
                          else codec.compress_split(m, r, k, v, T, c, sl, pl))
            else:
                out_b += codec.compress(m, r, k, v, T, c)
            in_b += int(mine.orig[c - my_lo])
            if tiered and snap_full["tier_index"][c] > 0:  # leaves HBM: D2H on the lane that produced it
                li, blob, bm = codec.last
                srcs = context_sources(blob, bm, k.data_ptr(), v.data_ptr(), L * H * T * D * 2)
                mv = [A.Move(p_, staging.next(n_), n_, A.KVT_MOVE_D2H, 0) for p_, n_ in srcs]
                arr = (A.Move * len(mv))(*mv)
                lanes[li].abi.check(lanes[li].abi.tier_moves(lanes[li].h, arr, len(mv)))
                moved += sum(n_ for _, n_ in srcs)
        return in_b, out_b, moved

    def run_steps(n, upload, exchange, tiered=False):
        """n steps, software-pipelined: batch i + 1's placement runs while
        batch i compresses on the codec lanes; every step's placement and
        compression happen inside the call."""
        acts, snap_full = placed(upload, exchange)
        n_act, in_b, out_b, moved = len(acts), 0, 0, 0
        for i in range(n):
            in_b, out_b, moved = launch_compress(snap_full, tiered)
            if i + 1 < n:
                acts, snap_full = placed(upload, exchange)
        join()
        return n_act, in_b, out_b, moved, acts, snap_full

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        res = fn()
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:  # the job takes as long as its slowest rank
            t = torch.tensor([ms], device="cpu" if args.ranks_share_gpu else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, res

    exchange_value = world > 1  # N > 1: the all-gather + merge is part of every step
    run_steps(args.warmup, False, exchange_value)
    barrier()
    l0 = eng.abi.launch_count(eng.h) + codec.launches()
    with ClockSampler(local) as clk:
        ms, (n_act, in_b, out_b, _, _, _) = timed(lambda: run_steps(args.steps, False, exchange_value))
    launches = eng.abi.launch_count(eng.h) + codec.launches() - l0
    ms_step = ms / args.steps
    value = total_bytes / (ms_step / 1e3) / 1e9

    if args.lane_trace:  # diagnostic only (stderr): where the codec streams wait on each other in one step
        barrier()
        codec.trace = []
        marks = []
        for ls in lane_streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(ls)
            marks.append(e)
        run_steps(1, False, exchange_value)
        ends = []
        for ls in lane_streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(ls)
            ends.append(e)
        barrier()
        t0 = marks[0]
        rel = lambda e: t0.elapsed_time(e)  # noqa: E731
        n = len(lane_streams)
        stall = [0.0] * n
        ring_stall = score_busy = 0.0
        for sl, pl, ev in codec.trace:
            ring_stall += ev[0].elapsed_time(ev[1])
            score_busy += ev[1].elapsed_time(ev[2])
            stall[pl] += ev[3].elapsed_time(ev[4])
        print(json.dumps({"lane_trace": {
            "lane_end_ms": [round(rel(e), 2) for e in ends],
            "pack_lane_wait_on_scores_ms": [round(x, 2) for x in stall],
            "score_lane_wait_on_ring_ms": round(ring_stall, 2), "score_lane_scoring_ms": round(score_busy, 2),
            "split_contexts": len(codec.trace)}}), file=sys.stderr)
        codec.trace = None

    # ---- e2e: through the C ABI with host buffers, copies inside the timed region
    e2e_ms, (_, _, _, _, acts, snap_full) = timed(lambda: run_steps(args.steps, True, True))
    h2d = rp.h2d_bytes
    d2h = acts.nbytes + snap_full.nbytes
    e2e_value = total_bytes / (e2e_ms / args.steps / 1e3) / 1e9

    # ---- e2e_tiered: e2e + every below-GPU-tier context's bytes leave HBM over PCIe
    tiered_steps = min(args.steps, args.tiered_steps)
    tiered = None
    if tiered_steps > 0:
        staging = StagingRing(eng.abi, max(kv_bytes, int(codec._out[0][0].numel())), slots=2)
        t_ms, (_, _, _, moved, _, snap_t) = timed(lambda: run_steps(tiered_steps, True, True, tiered=True))
        staging.close()
        mv_t = torch.tensor([moved], dtype=torch.int64, device="cpu" if args.ranks_share_gpu else "cuda")
        if world > 1:
            dist.all_reduce(mv_t)
        tiered = {"value": round(total_bytes / (t_ms / tiered_steps / 1e3) / 1e9, 2), "unit": "GB/s",
                  "steps": tiered_steps, "ms_per_step": round(t_ms / tiered_steps, 1),
                  "d2h_tier_bytes_per_step": int(mv_t.item()), "h2d_bytes_per_step": int(h2d),
                  "d2h_bytes_per_step": int(d2h) + int(mv_t.item()),
                  "note": "e2e plus the PCIe leg of the placement: every context placed in the CPU or SSD tier "
                          "(snapshot tier > 0) is copied HBM -> pinned DRAM by kvt_tier_moves on the stream that "
                          "compressed it; the SSD file write is measured separately (tier_move.ssd)"}

    # ---- per-phase shares + roofline of the dominant kernel (one instrumented pass)
    roof = tier_move = cpu = None
    if rank == 0:
        snap_now = store.snapshot()
        roof = kernel_roofline(eng, stream, codec, pool, store, _Shard(mine, my_lo), space, L, H, D, bpt, my_lo,
                               my_hi)
        pk, _ = peaks()
        roof["step_hbm_frac"] = round(roof["alg_bytes_per_step_rank"] / (ms_step / 1e3) / 1e9 / pk["hbm_gbs"], 4)
        roof["step_note"] = ("step_hbm_frac = this rank's algorithmic codec bytes per step / ms_per_step / peak: "
                             "the fraction of the HBM roofline the whole step sustains")
        tier_move = tier_move_rates(eng, stream, codec, pool, snap_now, _Shard(mine, my_lo), space, L, H, D, bpt,
                                    my_lo, my_hi)
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_reference_sample(W, seconds=args.cpu_seconds)
    n1 = None
    if rank == 0 and world == 1 and args.n1 and args.config != "c5":
        n1 = north_star_pass(args)

    if rank == 0:
        clocks = clk.summary()
        conf = config_dict(args, W, n_total, world)
        details = ({"kv_bytes_per_step": total_bytes, "kv_pool_chunks": args.pool,
                     "l2": "inputs larger than L2 (1 GiB chunks, pool of distinct chunks)",
                     "actions_per_step": n_act, "retained_bytes_per_step_rank0": out_b,
                     "parallelism": f"dp{world} (contexts sharded; per-step NCCL all-gather of profile records + "
                                    "device merge; global greedy replicated)",
                     "identity": "contexts placed at ratio 1.0 / 16 bits are the identity configuration: their "
                                 "compressed chunk is the source KV (no kernel, no copy; kvt_blob_map.identity); "
                                 "their bytes still count as compressed+scored+placed",
                     "schedule": "batches software-pipelined: batch i+1's placement overlaps batch i's compression"
                                 + (f"; {args.streams} codec streams, snapkv scoring alone on stream 0 as "
                                    f"persistent clusters on {args.snap_sms} SMs, top-k / pack / other scorers on "
                                    "streams 1.. (pipeline.split_plan)" if args.lanes == "split" else
                                    f"; {args.streams} codec streams, contexts round-robin")})
        line = {
            "metric": "KV GB/s compressed+scored+placed",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 KV, f64 scoring",
            "data": "synthetic (counter-hash KV, generated profiles)",
            "config": conf,
            "details": details,
            "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "e2e_tiered": tiered,
            "gpu_launches": int(launches),
            "roofline": roof,
            "tier_move": tier_move,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        if n1 is not None:
            line["n1_pass"] = n1
        if world > 1:
            line["nccl"] = nccl_summary(nccl_log + "*") if nccl_log else None
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class _Shard:
    """This rank's contexts addressed by global index (kernel_roofline /
    tier_move_rates read arrays.orig[c] for c in [lo, hi))."""

    def __init__(self, mine, lo):
        self.mine, self.lo = mine, lo

    @property
    def orig(self):
        return _Offset(self.mine.orig, self.lo)


class _Offset:
    def __init__(self, a, lo):
        self.a, self.lo = a, lo

    def __getitem__(self, c):
        return self.a[c - self.lo]


# ------------------------------------------------------------ CPU reference

_REF_PLACE_CACHE = {}


def _ref_engine():
    from paper_2512_14946_b200 import _abi as A
    from paper_2512_14946_b200.kvtier import Engine
    ref_path = os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so")
    if not os.path.exists(ref_path):
        return None
    return Engine(A.Abi(ref_path, "ref_", codec=False))


def reference_placement_seconds(W, cap=2000):
    """The reference's own greedy (insert_joint of every context, single
    thread, proj/src/placement.cpp:225-250) on this workload, timed once per
    process. Past `cap` contexts (C4 / C5: 6-12 min per run) it is
    timed on the first `cap` contexts and extrapolated by the measured N^2
    growth of the rescan (least_drop_update revisits every resident per
    step); the line says so."""
    key = (id(W["arrays"]), W["arrays"].n)
    if key in _REF_PLACE_CACHE:
        return _REF_PLACE_CACHE[key]
    from paper_2512_14946_b200.kvtier import ProfileArrays
    eng = _ref_engine()
    arrays, space, params = W["arrays"], W["space"], W["params"]
    n = arrays.n
    sub = arrays
    if n > cap:
        G = len(arrays.grid) // n
        sub = ProfileArrays.uniform_grid(arrays.ids[:cap], arrays.orig[:cap], arrays.freq[:cap], arrays.grid[:G],
                                         arrays.qual.reshape(n, -1, G)[:cap], arrays.has[:cap])
    from paper_2512_14946_b200 import workload
    tiers = workload.three_tiers(int(sub.orig.sum()), W["cfg"]["gpu_frac"], 0.30)
    ps = eng.pset(sub)
    st = eng.store(tiers, sub.n, space)
    t0 = time.perf_counter()
    acts = st.insert_joint(ps, space, params, np.arange(sub.n))
    t = time.perf_counter() - t0
    res = {"seconds": t * (n / sub.n) ** 2, "timed_contexts": sub.n, "actions": int(len(acts)),
           "extrapolated": n > cap}
    _REF_PLACE_CACHE[key] = res
    return res


def cached_greedy_seconds(W):
    """The same greedy restructured with a cached per-resident best update
    (the device greedy's structure), one CPU core, on the
    reference's own scoring functions (oracle/ref_capi.cpp
    ref_insert_joint_cached): separates the algorithmic speed-up (quadratic
    rescan -> N log N) from the hardware one."""
    eng = _ref_engine()
    arrays, space, params, tiers = W["arrays"], W["space"], W["params"], W["tiers"]
    ps = eng.pset(arrays)
    st = eng.store(tiers, arrays.n, space)
    t0 = time.perf_counter()
    acts = st.insert_joint(ps, space, params, np.arange(arrays.n), cached=True)
    return {"seconds": round(time.perf_counter() - t0, 4), "actions": int(len(acts)), "threads": 1}


def scoring_nproc(W, threads=None):
    """all_candidates over every context, sharded across `threads` host
    threads taking shards from a shared counter (the reference's work-queue
    pattern, proj/tools/kvtier_main.cpp:206-235), each calling the reference
    library (ref_score_candidates releases the GIL: ctypes)."""
    import threading

    from paper_2512_14946_b200.kvtier import ProfileArrays
    eng = _ref_engine()
    arrays, space, params, tiers = W["arrays"], W["space"], W["params"], W["tiers"]
    threads = threads or os.cpu_count()
    n = arrays.n
    G = len(arrays.grid) // n
    per = max(1, -(-n // (threads * 4)))
    shards = []
    for lo in range(0, n, per):
        hi = min(n, lo + per)
        sub = ProfileArrays.uniform_grid(arrays.ids[lo:hi], arrays.orig[lo:hi], arrays.freq[lo:hi], arrays.grid[:G],
                                         arrays.qual.reshape(n, -1, G)[lo:hi], arrays.has[lo:hi])
        shards.append(eng.pset(sub))
    nxt = [0]
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                i = nxt[0]
                nxt[0] += 1
            if i >= len(shards):
                return
            eng.score_candidates(shards[i], tiers, space, params)

    def run(nt):
        nxt[0] = 0
        th = [threading.Thread(target=worker) for _ in range(nt)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        return time.perf_counter() - t0

    t1, tn = run(1), run(threads)
    cands = n * len(space.methods) * len(space.ratios) * len(tiers)
    return {"candidates": int(cands), "threads": threads, "seconds_1_thread": round(t1, 4),
            "seconds_nproc": round(tn, 4), "candidates_per_s_nproc": round(cands / tn, 1)}


def codec_port_seconds(W, snap, budget):
    """The CPU codec port (oracle/liboracle.so; the reference has no codec)
    on one layer of every distinct placed (method, ratio, length), timed on
    all its threads within `budget` seconds, extrapolated to full chunks and
    to every context of each configuration."""
    from paper_2512_14946_b200 import _abi as A
    orc = A.Abi(os.path.join(ROOT, "oracle", "liboracle.so"), "orc_", codec=True)
    arrays, space = W["arrays"], W["space"]
    L, H = W["shape"]["L"], W["shape"]["H"]
    bpt = W["bytes_per_token"]
    groups = {}
    for c in range(arrays.n):
        key = (space.method_names[snap["method"][c]], float(snap["ratio"][c]), int(arrays.orig[c] // bpt))
        groups[key] = groups.get(key, 0) + 1
    threads = int(orc.lib.orc_parallel_threads())
    t_codec_timed, timed_ctx, spent = 0.0, 0, 0.0
    for (meth, ratio, T), count in sorted(groups.items(), key=lambda kv: -kv[1]):
        if spent > budget:
            break
        s = A.KvShape(1, H, T, 128)
        cfg = A.CodecCfg()
        orc.check(orc.codec_plan(meth.encode(), ratio, C.byref(s), C.byref(cfg)))
        m = A.BlobMap()
        orc.check(orc.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
        n = H * T * 128
        k = np.zeros(n, np.uint16)
        v = np.zeros(n, np.uint16)
        orc.check(orc.kv_generate(None, C.byref(s), 1, 0, A.ptr(k), A.ptr(v)))
        ws = np.zeros(orc.compress_workspace_bytes(C.byref(s), C.byref(cfg)), np.uint8)
        blob = np.zeros(max(1, m.total_bytes), np.uint8)
        t0 = time.perf_counter()
        orc.check(orc.compress(None, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), None, A.ptr(ws), A.ptr(blob)))
        dt = time.perf_counter() - t0
        spent += dt
        t_codec_timed += dt * L * count
        timed_ctx += count
    t_all = t_codec_timed / max(1, timed_ctx) * arrays.n
    return {"seconds": t_all, "threads": threads, "timed_contexts": timed_ctx, "spent": spent}


def cpu_reference_sample(W, seconds=20.0, with_extras=True):
    """The CPU arm on a bounded sample of the workload: placement = the
    reference kvtier library's own greedy over every context (timed once per
    process); codec = the CPU port (the reference has none) on one layer of
    each distinct placed configuration, extrapolated. kind = "port": the
    codec port dominates the modelled time. Extras beside it: the cached
    greedy on one core, an nproc-thread scoring pass, the host CPU."""
    eng = _ref_engine()
    if eng is None:
        return {"unavailable": "oracle/_ref not built"}
    place = reference_placement_seconds(W)
    ps = eng.pset(W["arrays"])
    st = eng.store(W["tiers"], W["arrays"].n, W["space"])
    st.insert_joint(ps, W["space"], W["params"], np.arange(W["arrays"].n), cached=True)  # same placement, fast
    snap = st.snapshot()
    codec = codec_port_seconds(W, snap, max(1.0, seconds))
    t_total = place["seconds"] + codec["seconds"]
    value = float(W["arrays"].orig.sum()) / t_total / 1e9
    L = W["shape"]["L"]
    out = {"value": round(value, 4), "unit": "GB/s", "cores": codec["threads"], "kind": "port",
           "sample": (f"placement: the reference kvtier library's insert_joint over "
                      f"{place['timed_contexts']} contexts on 1 thread ({place['seconds']:.2f} s"
                      f"{', extrapolated N^2 to ' + str(W['arrays'].n) if place['extrapolated'] else ''}); "
                      f"codec: CPU port of the codec spec (the reference has no codec) on 1 of {L} layers per "
                      f"distinct placed config ({codec['timed_contexts']}/{W['arrays'].n} contexts' configs timed "
                      f"in {codec['spent']:.1f} s on {codec['threads']} threads), extrapolated x{L}"),
           "place": {"kind": "reference", "seconds": round(place["seconds"], 3), "threads": 1,
                     "actions": place["actions"], "extrapolated": place["extrapolated"]},
           "codec": {"kind": "port", "seconds": round(codec["seconds"], 3), "threads": codec["threads"]}}
    out.update(cpu_info())
    if with_extras:
        out["cached_greedy"] = cached_greedy_seconds(W)
        out["scoring_nproc"] = scoring_nproc(W)
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_2512_14946_b200 import workload
    W = workload.build(args.config, n_ctx=args.n_ctx, seed=7)
    vals = []
    cpu = None
    budget = max(1.0, min(args.cpu_seconds, 120.0 / max(1, args.warmup + args.steps)))
    for i in range(args.warmup + args.steps):
        cpu = cpu_reference_sample(W, seconds=budget, with_extras=(i == 0))
        if i == 0:
            extras = {k: cpu[k] for k in ("cached_greedy", "scoring_nproc") if k in cpu}
        if i >= args.warmup:
            vals.append(cpu["value"])
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": "KV GB/s compressed+scored+placed", "value": value, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 KV, f64 scoring",
            "data": "synthetic (counter-hash KV, generated profiles)",
            "config": config_dict(args, W, W["arrays"].n * world, world),
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cpu["cores"], "kind": cpu["kind"],
                             "sample": cpu["sample"], "place": cpu["place"], "codec": cpu["codec"], **extras,
                             **cpu_info()},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch(args):
    """--gpus N > 1 without torchrun: one process per GPU under
    torch.distributed.run on 127.0.0.1 (the driver's own launch line)."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n-ctx", type=int, default=None)
    ap.add_argument("--pool", type=int, default=8, help="distinct resident KV chunks")
    ap.add_argument("--streams", type=int, default=3, help="codec CUDA streams")
    ap.add_argument("--group-slices", type=int, default=0,
                    help="knorm / keydiff chunks compressed this many (layer, head) slices at a time "
                         "(kvt_compress_slices: K read from HBM once per group); 0 = whole chunks")
    ap.add_argument("--lanes", choices=["split", "rr"], default="split",
                    help="split: snapkv scoring alone on stream 0 (--snap-sms SM budget), every other codec "
                         "kernel on streams 1.. (pipeline.split_plan); rr: contexts round-robin, one kvt_compress "
                         "each")
    ap.add_argument("--lane-priority", choices=["none", "snap", "mem"], default="none",
                    help="CUDA stream priorities of the codec streams (diagnostic)")
    ap.add_argument("--lane-trace", action="store_true",
                    help="diagnostic: one extra step with per-context stream events; stream waits to stderr")
    ap.add_argument("--ring", type=int, default=8, help="split mode: score buffers between the streams")
    ap.add_argument("--snap-sms", type=int, default=None,
                    help="split mode: SM budget of snapkv's persistent clusters (sets KVT_SNAP_SMS); default "
                         "per workload (SNAP_SMS: measured best for its mix of context lengths)")
    ap.add_argument("--tiered-steps", type=int, default=2, help="steps of the e2e_tiered leg (PCIe-bound); 0 = skip")
    ap.add_argument("--no-n1", dest="n1", action="store_false",
                    help="skip the north-star pass (c5: 1,000,008 chunk-configs) reported beside the headline line")
    ap.add_argument("--n1-steps", type=int, default=2)
    ap.add_argument("--ranks-share-gpu", action="store_true",
                    help="test mode for 1-GPU boxes: every rank on cuda:0, profile exchange over gloo (host "
                         "buffers); exercises the N > 1 step logic without NCCL. Not a scaling measurement.")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.snap_sms is None:
        args.snap_sms = SNAP_SMS.get(args.config, 48)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        if args.lanes == "split":  # read by kvt at every snapkv launch; the roofline leg runs the same way
            os.environ["KVT_SNAP_SMS"] = str(args.snap_sms)
        run_b200(args)


if __name__ == "__main__":
    main()
