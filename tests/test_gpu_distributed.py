"""Device side of the multi-GPU profile exchange: kvt_pset_merge over
gathered rank records (what NCCL's all-gather hands every rank) builds the
same profile set as pset_create on the concatenated rows — every candidate
table and the greedy's action list identical — and refills in place."""
import numpy as np
import pytest
import torch

from paper_2512_14946_b200 import distributed, workload
from paper_2512_14946_b200.kvtier import Engine, MergedPSet

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,config", [(1, "c2"), (3, "c3"), (8, "c1")])
def test_gpu_pset_merge_equals_pset_create(gpu_abi, world, config):
    eng = Engine(gpu_abi)
    n = 50
    Ws = [workload.build(config, n_ctx=n, seed=7 + r) for r in range(world)]
    recs = np.concatenate([distributed.pack_record(eng.abi, w["arrays"]) for w in Ws])
    M, g = Ws[0]["arrays"].M, int(Ws[0]["arrays"].goff[-1])
    dev = torch.from_numpy(recs).cuda()
    ps = MergedPSet(eng, world * n).merge(dev, world, n, g, M)
    cat = distributed.merge_rank_profiles([w["arrays"] for w in Ws])
    ref = eng.pset(cat)
    tiers = workload.three_tiers(int(cat.orig.sum()), Ws[0]["cfg"]["gpu_frac"], 0.3)
    a = eng.score_candidates(ps, tiers, Ws[0]["space"], Ws[0]["params"])
    b = eng.score_candidates(ref, tiers, Ws[0]["space"], Ws[0]["params"])
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    runs = []
    for p in (ps, ref):
        st = eng.store(tiers, cat.n, Ws[0]["space"])
        runs.append(st.insert_joint(p, Ws[0]["space"], Ws[0]["params"], np.arange(cat.n)))
    assert np.array_equal(runs[0], runs[1]) and len(runs[0]) >= cat.n
    # refill in place with other rows: the set follows (new id, no stale tables)
    Ws2 = [workload.build(config, n_ctx=n, seed=70 + r) for r in range(world)]
    dev.copy_(torch.from_numpy(np.concatenate([distributed.pack_record(eng.abi, w["arrays"]) for w in Ws2])))
    p_before = ps.p.value
    ps.merge(dev, world, n, g, M)
    assert ps.p.value == p_before
    cat2 = distributed.merge_rank_profiles([w["arrays"] for w in Ws2])
    c = eng.score_candidates(ps, tiers, Ws[0]["space"], Ws[0]["params"])
    d = eng.score_candidates(eng.pset(cat2), tiers, Ws[0]["space"], Ws[0]["params"])
    for k in c:
        assert np.array_equal(c[k], d[k]), k
