# Memory-bound codec kernels with B SMs held by a spinning blocker kernel (scores
# + pack of a full chunk per method): GB/s and GB/s per free SM. Build the
# blocker first: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared
# -Xcompiler -fPIC profiles/sm_blocker.cu -o profiles/libsm_blocker.so
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_14946_b200 as pkg
from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import Engine
blk = C.CDLL(os.path.abspath("profiles/libsm_blocker.so"))
s2 = torch.cuda.Stream()
eng = Engine(pkg.product(), stream=s2.cuda_stream)
ab = eng.abi
s = A.KvShape(32, 8, 8192, 128)
n = s.L * s.H * s.T * s.D
k = torch.empty(n, dtype=torch.int16, device="cuda"); v = torch.empty_like(k)
ab.check(ab.kv_generate(eng.h, C.byref(s), 1, 0, A.ptr(k), A.ptr(v)))
torch.cuda.synchronize()
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
bs = torch.cuda.Stream()
for spec in ["knorm-q4:0.2", "knorm-q8:0.6", "knorm:0.4"]:
    meth, ratio = spec.split(":")
    cfg = A.CodecCfg(); ab.check(ab.codec_plan(meth.encode(), float(ratio), C.byref(s), C.byref(cfg)))
    m = A.BlobMap(); ab.check(ab.blob_layout(C.byref(s), C.byref(cfg), C.byref(m)))
    S = s.L * s.H
    sc = torch.empty(S * s.T, dtype=torch.float32, device="cuda")
    idx = torch.zeros(S * cfg.keep, dtype=torch.int32, device="cuda")
    blob = torch.empty(m.total_bytes, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(s2):
        ab.check(ab.token_scores(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(sc)))
        ab.check(ab.topk(eng.h, C.byref(s), C.byref(cfg), A.ptr(sc), A.ptr(idx)))
    torch.cuda.synchronize()
    kk = cfg.keep
    alg = {"scores": S * s.T * 260, "pack": 2 * S * kk * 256 + m.total_bytes}
    for nb in [0, 24, 48, 72]:
        res = {}
        for ph in ("scores", "pack"):
            times = []
            for rep in range(4):
                flag.zero_()
                torch.cuda.synchronize()
                if nb:
                    blk.blocker_launch(C.c_void_p(bs.cuda_stream), nb, C.c_void_p(flag.data_ptr()))
                    time.sleep(0.002)
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s2)
                if ph == "scores":
                    ab.check(ab.token_scores(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), None, A.ptr(sc)))
                else:
                    ab.check(ab.pack(eng.h, C.byref(s), C.byref(cfg), A.ptr(k), A.ptr(v), A.ptr(idx), A.ptr(blob)))
                e1.record(s2)
                e1.synchronize()
                flag.fill_(1)
                torch.cuda.synchronize()
                if rep: times.append(e0.elapsed_time(e1))
            ms = sorted(times)[len(times) // 2]
            gbs = alg[ph] / (ms / 1e3) / 1e9
            res[ph] = (round(ms, 4), round(gbs), round(gbs / (148 - nb)))
        print(json.dumps({"method": spec, "blocked_sms": nb, "ms_GBps_perSM": res}), flush=True)
