"""GPU parity of the batched forward-staging plan (csrc/k_stage.cu) against the
oracle composition of fire_prefetch's target choice (engine.cpp:1137-1166) and
on_prefetch_requested (manager.cpp:60-100): target, action kind, skip reason, [from, to)."""
import numpy as np
import pytest
import torch

from batch_oracle import apply_warm_gpu, apply_warm_oracle, warm_ops
from oracle.py_oracle import Restated

pytestmark = pytest.mark.gpu


def test_stage_plan_matches_oracle():
    import ctypes as C
    from paper_2604_25899_b200 import Context, _lib
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import workload as W
    B = 16
    tr = W.deep_research(n_workflows=30, seed=12, device="cpu")
    cl = W.make_cluster(9, 2, kv=40_000, l2=40_000, seed=3, interleave=True)
    o = Restated(B)
    caches = [o.new_cache(int(cl.kv_capacity[n]), int(cl.l2_capacity[n])) for n in range(9)]
    l3, reg = o.new_l3(), o.new_registry()
    ctx = Context(9, cl.kv_capacity, cl.l2_capacity, B)
    ops = warm_ops(tr, cl, 4, n_chains=8)
    apply_warm_oracle(o, caches, l3, reg, tr, ops)
    apply_warm_gpu(ctx, tr, ops)
    rng = np.random.default_rng(2)
    # successor prefixes: cuts of the burst's prompts (some empty, some full, some ragged)
    idx = rng.choice(tr.R, 200, replace=False)
    prefixes = []
    for r in idx:
        p = tr.prompt(int(r))
        cut = int(rng.choice([0, len(p), rng.integers(0, len(p) + 1)]))
        prefixes.append(p[:cut])
    off = np.zeros(len(prefixes) + 1, np.int64)
    np.cumsum([len(p) for p in prefixes], out=off[1:])
    toks = np.concatenate(prefixes) if off[-1] else np.zeros(1, np.uint64)
    grp = tr.group[idx].astype(np.int32)
    res = np.zeros(len(prefixes), PB.RES_DTYPE)
    db = PB.upload_batch(ctx, toks, off, res, grp, grp, grp)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand)
    idle = rng.integers(0, 2, 9).astype(np.int8)
    d_idle = torch.from_numpy(idle).cuda()
    out = torch.zeros((len(prefixes), 4), dtype=torch.int64, device="cuda")
    PB.bind_current_stream(ctx)
    PB.hash_batch(ctx, db)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib._lib.pyg_stage_plan_dev(ctx.h, p(db.tokens), p(db.tok_off), p(db.hash_off),
                                            p(db.hashes), len(prefixes), p(db.group), dn.n_groups,
                                            p(dn.cand_off), p(dn.cand), dn.max_cand,
                                            p(dn.replica_id), p(d_idle), p(out)))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    kinds = {"promote": 0, "background": 1, "skip": 2}
    seen = set()
    for k, pre in enumerate(prefixes):
        g = int(grp[k])
        cands = cl.cand[cl.cand_off[g]:cl.cand_off[g + 1]]
        best, best_l2 = -1, -1
        for n in cands:
            l2 = o.lookup(caches[n], None, pre)[1] if len(pre) else 0
            if best < 0 or l2 > best_l2 or (l2 == best_l2 and cl.replica_id[n] < cl.replica_id[best]):
                best, best_l2 = int(n), l2
        m = o.lookup(caches[best], l3, pre)
        staged = max(m[0], m[1])
        if len(pre) == 0:
            want = (best, kinds["skip"], 1, 0, 0)
        elif staged >= len(pre):
            want = (best, kinds["skip"], 2, 0, 0)
        elif m[2] > staged:
            want = (best, kinds["promote"], 0, staged, m[2])
        elif idle[best]:
            want = (best, kinds["background"], 0, staged, len(pre))
        else:
            want = (best, kinds["skip"], 3, 0, 0)
        row = got[k]
        tgt, kind, reason = int(row[0] & 0xffffffff), int(row[0] >> 32), int(row[1] & 0xffffffff)
        assert (tgt, kind, reason, int(row[2]), int(row[3])) == want, k
        seen.add(want[1:3])
    assert len(seen) >= 3  # several action kinds exercised
