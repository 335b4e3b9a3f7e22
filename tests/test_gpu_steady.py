"""The steady-state burst sequence (paper_2604_25899_b200/steady.py, the bench workload)
against the unmodified reference driven through the same sequence (oracle/steady_ref.py):
per burst the staged matrix, every decision (target, tiebreak, headroom, oom_bound bits),
admissions and lookups; at the end every replica's L1/L2 and the shared L3, record for
record.  The cluster carries state across bursts (placements held for two bursts, releases,
L1 near full so admissions evict, L3 promotions in engine order)."""
import numpy as np
import pytest
import torch

from oracle.py_oracle import reference_available


def _scenario(B, n_bursts, R, n_rep, n_models, kv, seed):
    from paper_2604_25899_b200 import steady as S
    from paper_2604_25899_b200 import workload as W
    kw = dict(mean_len=500, n_prefixes=24)
    bursts = S.make_bursts(n_bursts, R, seed=seed, device="cpu", n_models=n_models, **kw)
    warm = W.bursty(n_requests=4 * R, seed=seed + 77, device="cpu", n_models=n_models,
                    r_base=10_000_000, **kw)
    cl = W.make_cluster(n_rep, n_models, kv=kv, l2=kv, seed=seed)
    ops = S.warm_ops(warm, cl, l3_prefixes=16, l2_per_group=8, seed=seed)
    off, placed = S.warm_fill_plan(warm, cl, fill_frac=0.97)
    return bursts, warm, cl, ops, off, placed


def _ref_run(B, bursts, warm, cl, ops, off, placed):
    from oracle.steady_ref import RefSteady
    from paper_2604_25899_b200 import steady as S
    ref = RefSteady(B, cl, threads=4)
    ref.warm(warm, ops, off, placed)
    outs = []
    for k, tr in enumerate(bursts):
        rw, rm = S.registry_pairs(tr.wf, tr.role)
        outs.append(ref.step(k, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role,
                             rw, rm, 1.0 + k, S.hold_of(k, tr.R, tr.R), want_staged=True))
    return ref, outs


@pytest.mark.skipif(not reference_available(16), reason="oracle/_ref not built")
def test_steady_reference_sequence_evicts_and_places():
    """CPU: the reference side of the sequence places, admits and evicts (so the GPU parity
    test below covers eviction, holds and releases)."""
    bursts, warm, cl, ops, off, placed = _scenario(16, 4, 300, 12, 3, 20_000, 3)
    ref, outs = _ref_run(16, bursts, warm, cl, ops, off, placed)
    placed_n = sum(int((d["target"] >= 0).sum()) for d, _, _, _ in outs)
    admitted = sum(int(a.sum()) for _, a, _, _ in outs)
    assert placed_n > 20 and admitted > 10
    # L1 near full: occupancy close to capacity on most replicas
    occ = [ref.ref.occupancy(ref.caches[n], None, 0) for n in range(cl.n_replicas)]
    assert sum(o > 0.5 * cl.kv_capacity[0] for o in occ) >= cl.n_replicas // 2


@pytest.mark.gpu
@pytest.mark.parametrize("B,seed", [(16, 1), (16, 2), (64, 3)])
def test_steady_sequence_matches_reference(B, seed):
    if not reference_available(B):
        pytest.skip("oracle/_ref not built")
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import steady as S
    bursts, warm, cl, ops, off, placed = _scenario(B, 5, 400, 16, 4, 24_000, seed)
    ref, want = _ref_run(B, bursts, warm, cl, ops, off, placed)
    dev = torch.device("cuda", 0)
    ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, B)
    assert S.apply_warm_fill_gpu(ctx, warm, off, placed, B, dev) == len(placed)
    S.apply_ops_gpu(ctx, warm, ops)
    db = [S.upload_burst(tr, B, dev, k) for k, tr in enumerate(bursts)]
    st = S.Steady(ctx, cl, max(b.R for b in db), dev)
    ctx.counters(reset=True)
    for k in range(len(db)):
        PB.bind_current_stream(ctx)
        PB.hash_batch(ctx, db[k].b)
        o = st.step(k, db, 1.0 + k)
        torch.cuda.synchronize()
        ctx.check_device_error()
        got = o.host()
        R = db[k].R
        d, a, m3, stg = want[k]
        mc = stg.shape[1]
        assert np.array_equal(got["staged"][:R, :mc], stg), k
        assert np.array_equal(got["decisions"][:R]["target"], d["target"]), k
        assert np.array_equal(got["decisions"][:R]["tiebreak"], d["tiebreak"]), k
        assert np.array_equal(got["decisions"][:R]["headroom"], d["headroom"]), k
        assert got["decisions"][:R]["oom_bound"].tobytes() == d["oom_bound"].tobytes(), k
        assert np.array_equal(got["admitted"][:R], a), k
        pl = d["target"] >= 0
        assert np.array_equal(got["match3"][:R][pl], m3[pl]), k
    for n in range(cl.n_replicas):
        for t in (0, 1):
            assert ctx.dump(n, t).tobytes() == ref.dump(n, t).tobytes(), (n, t)
    assert ctx.dump(0, 2).tobytes() == ref.dump(0, 2).tobytes()
    assert ctx.counters()["evicted_blocks"] > 0
