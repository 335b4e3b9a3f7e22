"""Golden vectors produced by the reference itself (tests/golden/make_golden.py over
oracle/_ref).  CPU: the C restatement reproduces every one.  GPU (-m gpu): the CUDA
path reproduces every one.  Nothing here needs /root/reference at run time."""
import gzip
import json
import os

import numpy as np
import pytest

import test_oracle as T
from oracle.py_oracle import Restated
from oracle.step import apply_warm_gpu, apply_warm_oracle, oracle_step, warm_ops

G = json.load(gzip.open(os.path.join(os.path.dirname(__file__), "golden",
                                     "reference_golden.json.gz"), "rt"))


def dec(x):
    if isinstance(x, dict) and "b" in x:
        return bytes.fromhex(x["b"])
    if isinstance(x, dict) and "f" in x:
        return float.fromhex(x["f"])
    if isinstance(x, list):
        return [dec(v) for v in x]
    return x


def _norm(v):
    if isinstance(v, (list, tuple)):
        return [_norm(x) for x in v]
    if isinstance(v, (np.integer,)):
        return int(v)
    if isinstance(v, (np.floating,)):
        return float(v)
    if isinstance(v, bool):
        return int(v)
    return v


def check_backend(make):
    for B in ("16", "64"):
        be = make(int(B))
        for case in G["hashes"][B]:
            t = np.array(case["tokens"], np.uint64)
            assert be.chain_hashes(t).tolist() == case["hashes"]
        for seed, transcript in G["ops"][B].items():
            got = T._random_ops(be, int(seed), int(B), n_ops=120)
            assert _norm(got) == _norm(dec(transcript))
    be = make(16)
    for rc in G["routes"]:
        spec = [(a, b, [tuple(x) for x in c], d) for a, b, c, d in rc["spec"]]
        assert list(T.route(be, spec, tuple(rc["req"]))) == dec(rc["decision"])


def test_restated_reproduces_reference_golden():
    check_backend(lambda B: Restated(B))


def test_restated_batch_steps_reproduce_reference_golden():
    from paper_2604_25899_b200 import workload as W
    for B, g in G["steps"].items():
        o = Restated(int(B))
        tr = W.deep_research(n_workflows=g["workflows"], seed=g["seed"], device="cpu")
        n, m, kv, l2, cseed = g["cluster"]
        cl = W.make_cluster(n, m, kv=kv, l2=l2, seed=cseed)
        caches = [o.new_cache(kv, l2) for _ in range(n)]
        l3, reg = o.new_l3(), o.new_registry()
        apply_warm_oracle(o, caches, l3, reg, tr, warm_ops(tr, cl, g["warm_seed"]))
        for s, st in enumerate(g["steps"]):
            got = oracle_step(o, caches, l3, reg, tr, cl, st["mode"], 0.05, 3.0 + s, True, True)
            assert _norm(got["decisions"]) == _norm(dec(st["decisions"]))
            assert got["placed"] == st["placed"]
            assert got["admitted"].tolist() == st["admitted"]
            dumps = [o.dump(c, None, t).tobytes().hex() for c in caches for t in (0, 1)]
            dumps.append(o.dump(caches[0], l3, 2).tobytes().hex())
            assert dumps == st["dumps"]


@pytest.mark.gpu
def test_gpu_reproduces_reference_golden():
    from backends import Gpu
    check_backend(lambda B: Gpu(B))


@pytest.mark.gpu
def test_gpu_batch_steps_reproduce_reference_golden():
    import torch
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import workload as W
    for B, g in G["steps"].items():
        tr = W.deep_research(n_workflows=g["workflows"], seed=g["seed"], device="cpu")
        n, m, kv, l2, cseed = g["cluster"]
        cl = W.make_cluster(n, m, kv=kv, l2=l2, seed=cseed)
        ctx = Context(n, kv, l2, int(B))
        apply_warm_gpu(ctx, tr, warm_ops(tr, cl, g["warm_seed"]))
        db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role)
        dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off,
                             cl.cand)
        out = PB.alloc_out(ctx, db, dn)
        for s, st in enumerate(g["steps"]):
            PB.step(ctx, db, dn, out, 3.0 + s, mode=st["mode"])
            torch.cuda.synchronize()
            h = out.host()
            d = h["decisions"][:tr.R]
            want = dec(st["decisions"])
            for r in range(tr.R):
                assert [int(d["target"][r]), int(d["tiebreak"][r]), int(d["headroom"][r]),
                        float(d["oom_bound"][r])] == list(want[r])
            po = h["placed_off"]
            assert [h["placed"][po[k]:po[k + 1]].tolist() for k in range(n)] == st["placed"]
            assert h["admitted"][:tr.R].tolist() == st["admitted"]
            dumps = [ctx.dump(k, t).tobytes().hex() for k in range(n) for t in (0, 1)]
            dumps.append(ctx.dump(0, 2).tobytes().hex())
            assert dumps == st["dumps"]
