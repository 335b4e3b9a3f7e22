"""The batched-step oracle composition itself (CPU): seq-commit spreads a burst
exactly like the engine's sequential route_request, snapshot herds it, and the
restated composition equals the reference library's on the same state."""
import numpy as np
import pytest

from batch_oracle import SEQ_COMMIT, SNAPSHOT, apply_warm_oracle, oracle_step, warm_ops
from oracle.py_oracle import Restated, Reference, reference_available
from paper_2604_25899_b200 import workload as W


def _state(o, tr, cl, seed=0):
    caches = [o.new_cache(int(cl.kv_capacity[n]), int(cl.l2_capacity[n]))
              for n in range(cl.n_replicas)]
    l3, reg = o.new_l3(), o.new_registry()
    apply_warm_oracle(o, caches, l3, reg, tr, warm_ops(tr, cl, seed))
    return caches, l3, reg


def test_seq_commit_spreads_snapshot_herds():
    """16 identical requests vs 4 empty nodes -> snapshot 0x16, seq 0,1,2,3,..."""
    o = Restated(16)
    tr = W.deep_research(n_workflows=2, seed=1, device="cpu").subset([0] * 16)
    tr.res["alpha"] = 1 - 0.99
    cl = W.make_cluster(4, 1, kv=10**9, l2=10**6, max_bg=0)
    tr.group[:] = 0
    for mode, expect in [(SNAPSHOT, [0] * 16), (SEQ_COMMIT, [0, 1, 2, 3] * 4)]:
        caches, l3, reg = _state(o, tr, cl)
        out = oracle_step(o, caches, l3, reg, tr, cl, mode, 0.05, 1.0, True, True)
        assert [d[0] for d in out["decisions"]] == expect


@pytest.mark.skipif(not reference_available(16), reason="oracle/_ref not built")
def test_step_restated_equals_reference():
    o, ref = Restated(16), Reference(16)
    tr = W.deep_research(n_workflows=10, seed=4, device="cpu")
    cl = W.make_cluster(6, 2, kv=20_000, l2=20_000, seed=5)
    outs = []
    for be in (o, ref):
        caches, l3, reg = _state(be, tr, cl)
        res = [oracle_step(be, caches, l3, reg, tr, cl, SEQ_COMMIT, 0.05, 5.0 + s, True, True)
               for s in range(2)]
        dumps = [be.dump(c, None, t).tobytes() for c in caches for t in (0, 1)]
        dumps.append(be.dump(caches[0], l3, 2).tobytes())
        outs.append((res, dumps))
    (ra, da), (rb, db) = outs
    for x, y in zip(ra, rb):
        assert x["decisions"] == y["decisions"]
        assert np.array_equal(x["staged"], y["staged"])
        assert x["placed"] == y["placed"]
        assert np.array_equal(x["admitted"], y["admitted"])
        assert np.array_equal(x["match3"], y["match3"])
    assert da == db


@pytest.mark.skipif(not reference_available(16), reason="oracle/_ref not built")
def test_reference_cpp_step_equals_composition():
    """pref_step (the CPU baseline, C++ over the reference) == the Python composition."""
    ref = Reference(16)
    tr = W.deep_research(n_workflows=10, seed=6, device="cpu")
    cl = W.make_cluster(6, 2, kv=20_000, l2=20_000, seed=7)
    c1, l1, g1 = _state(ref, tr, cl)
    c2, l2, g2 = _state(ref, tr, cl)
    for s in range(2):
        a = oracle_step(ref, c1, l1, g1, tr, cl, SEQ_COMMIT, 0.05, 5.0 + s, True, True)
        n, dec, adm = ref.step(c2, l2, g2, True, tr.tokens_np(), tr.tok_off, tr.res, tr.group,
                               tr.wf, tr.role, cl, SEQ_COMMIT, 0.05, 5.0 + s, True)
        assert [tuple(x) for x in dec.tolist()] == [tuple(d) for d in a["decisions"]]
        assert np.array_equal(adm, a["admitted"])
        assert n == sum(len(p) for p in a["placed"])
    for x, y in zip(c1, c2):
        for t in (0, 1):
            assert ref.dump(x, None, t).tobytes() == ref.dump(y, None, t).tobytes()
    assert ref.dump(c1[0], l1, 2).tobytes() == ref.dump(c2[0], l2, 2).tobytes()
