import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, ctypes as C
import paper_2512_14946_b200 as pkg
from paper_2512_14946_b200 import _abi as A
from paper_2512_14946_b200.kvtier import Engine
from test_gpu_codec import gen, scores, plan
import codec_ref as R
gpu = Engine(pkg.product()); orc = Engine(A.Abi("/root/repo/oracle/liboracle.so", "orc_", codec=True))
s = A.KvShape(2, 2, 300, 128)
kg, _ = gen(gpu, s); ko, _ = gen(orc, s, on_gpu=False)
cfg = plan(orc.abi, "keydiff", 0.3, s)
sg, so = scores(gpu, s, cfg, kg, True), scores(orc, s, cfg, ko, False)
sn = R.keydiff_scores(ko.reshape(2, 2, 300, 128)).reshape(-1)
bad = np.nonzero(sg.view(np.uint32) != so.view(np.uint32))[0]
print("mismatch", len(bad), "of", sg.size, "oracle==numpy", np.array_equal(so.view(np.uint32), sn.view(np.uint32)))
print(bad[:20]); print(sg[bad[:5]], so[bad[:5]])
print("rel", np.abs((sg - so) / so)[bad].max() if len(bad) else 0)
sg2 = scores(gpu, s, cfg, kg, True)
print("deterministic", np.array_equal(sg, sg2))
# hypotheses about S: recompute scores in numpy from variants of the sum
x = R.bf2f(ko.reshape(2, 2, 300, 128))
n2 = R.row_dot32(x, x)
inv = (np.float32(1) / np.sqrt(n2).astype(np.float32)).astype(np.float32)
def score_from_S(S):
    sd = (S.astype(np.float32) * np.float32(2.0 ** -21)).astype(np.float32)
    return (-(R.row_dot32(x, sd) * inv).astype(np.float32)).reshape(-1)
c = (inv * np.float32(2.0 ** 21)).astype(np.float32)
f = np.rint((x * c[..., None]).astype(np.float32)).astype(np.int64)
S = f.sum(-2, keepdims=True)
print("numpy S score==gpu", np.array_equal(score_from_S(S), sg))
for dS in (1, -1):
    for d in range(128):
        S2 = S.copy(); S2[..., d] += dS
        if np.array_equal(score_from_S(S2)[:300], sg[:300]):
            print("single-channel offset", d, dS)
# f without last token / first token
for drop in (0, 299):
    S3 = S - f[..., drop:drop + 1, :]
    print("drop", drop, np.sum(score_from_S(S3) != sg))
