"""Ordered L3 promotion in batched admission (engine.cpp:799-829 run one request at a
time): a later admission must not see the L3 spans an earlier one promoted
(erase_chain_span(L3, max(l1,l2), reusable), engine.cpp:826-828).

The chain scenario makes every admission depend on the one before it: replica n
holds the first 3*(K-1-n) blocks of a shared 40-block chain in L1, so admission n
promotes blocks [3*(K-1-n), x) where x is where admission n-1's promotion starts.
That is a dependency chain K deep: the device solves it with Jacobi rounds and
finishes it with the in-order fixup.  The oracle is the sequential composition
(oracle/step.py), pinned to the reference by tests/golden."""
import numpy as np
import pytest
import torch

from batch_oracle import SEQ_COMMIT, apply_warm_oracle, oracle_step
from oracle.py_oracle import Restated

K = 12          # replicas of model 0; replica K (model 1) holds the chain for the L3 write
CHAIN = 40      # blocks


def chain_scenario(B, n_extra=0, seed=0):
    from paper_2604_25899_b200 import workload as W
    rng = np.random.default_rng(seed)
    base = rng.integers(1, 1 << 62, size=CHAIN * B, dtype=np.uint64)
    prompts = []
    for r in range(K + 1 + n_extra):
        sfx = rng.integers(1, 1 << 62, size=3 * B + 5, dtype=np.uint64)
        prompts.append(np.concatenate([base, sfx]))
    lens = np.array([len(p) for p in prompts], np.int64)
    off = np.zeros(len(prompts) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = np.concatenate(prompts)
    R = len(prompts)
    res = np.zeros(R, W.RES_DTYPE)
    res["prompt_len"] = lens
    res["upper"] = 100
    res["alpha"] = 0.0
    group = np.zeros(R, np.int32)
    group[K] = 1                      # the chain carrier routes to replica K
    wf = np.arange(R, dtype=np.int32)
    wf[K] = 999
    role = np.ones(R, np.int32)
    tr = W.Trace(torch.from_numpy(toks.view(np.int64)), off, res, group, wf, role)
    n = K + 1
    cl = W.Cluster(n, np.array([0] * K + [1], np.int32), np.arange(n, dtype=np.int32),
                   np.full(n, 10_000_000, np.int64), np.full(n, 10_000_000, np.int64),
                   np.zeros(n + 1, np.int64), np.zeros(0, W.RES_DTYPE),
                   np.array([0, K, K + 1], np.int32), np.arange(n, dtype=np.int32))
    ops = []
    # the shared chain into replica K's L2 under workflow 999, role 1, then the completion
    # sweep writes it to L3 (RetainAndWriteL3, manager.cpp:44-58)
    ops.append(("ins", K, 1, K, CHAIN * B, 999, 1, 0.5, 0))
    ops.append(("cmp", 999, 0b10, 1.0))
    # replica n holds the first 3*(K-1-n) chain blocks in L1 (decreasing with n)
    for r in range(K):
        if K - 1 - r > 0:
            ops.append(("ins", r, 0, r, 3 * (K - 1 - r) * B, 500 + r, 2, 0.25, 0))
    for w in list(range(R)) + [999] + [500 + r for r in range(K)]:
        ops.append(("reg", w, 0b110))
    return tr, cl, ops


def _oracle(B, tr, cl, ops):
    o = Restated(B)
    caches = [o.new_cache(int(cl.kv_capacity[n]), int(cl.l2_capacity[n]))
              for n in range(cl.n_replicas)]
    l3, reg = o.new_l3(), o.new_registry()
    apply_warm_oracle(o, caches, l3, reg, tr, ops)
    return o, caches, l3, reg


@pytest.mark.parametrize("B", [16, 64])
def test_chain_scenario_oracle_is_a_chain(B):
    """CPU: the sequential oracle produces the dependency chain the GPU test relies on."""
    tr, cl, ops = chain_scenario(B)
    o, caches, l3, reg = _oracle(B, tr, cl, ops)
    want = oracle_step(o, caches, l3, reg, tr, cl, SEQ_COMMIT, 0.05, 3.0, True, True)
    tgt = [d[0] for d in want["decisions"]]
    assert tgt[:K] == list(range(K)) and tgt[K] == K
    l3m = [int(want["match3"][r][2]) for r in range(K)]
    # admission 0 (replica 0: L1 has 3(K-1) blocks) promotes the chain's tail; each later
    # one sees the chain cut where the previous promotion started
    assert l3m[0] == CHAIN * B
    for n in range(1, K):
        assert l3m[n] == 3 * (K - n) * B, (n, l3m)



@pytest.mark.gpu
@pytest.mark.parametrize("B", [16, 64])
def test_l3_promotion_chain_gpu(B):
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from test_gpu_batch import _compare_state
    from oracle.step import apply_warm_gpu
    tr, cl, ops = chain_scenario(B, n_extra=0, seed=B)
    o, caches, l3, reg = _oracle(B, tr, cl, ops)
    ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, B)
    apply_warm_gpu(ctx, tr, ops)
    db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand)
    out = PB.alloc_out(ctx, db, dn)
    PB.step(ctx, db, dn, out, 3.0)
    torch.cuda.synchronize()
    ctx.check_device_error()
    got = out.host()
    want = oracle_step(o, caches, l3, reg, tr, cl, SEQ_COMMIT, 0.05, 3.0, True, True)
    assert [int(x) for x in got["decisions"]["target"][:tr.R]] == [d[0] for d in want["decisions"]]
    assert np.array_equal(got["admitted"][:tr.R], want["admitted"])
    assert np.array_equal(got["match3"][:tr.R], want["match3"]), (got["match3"][:tr.R, 2],
                                                                   want["match3"][:, 2])
    _compare_state(o, caches, l3, ctx, cl)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_l3_shared_prefix_bursts_gpu(seed):
    """Random bursts over a few L3-resident chains shared by many requests on many replicas,
    several steps: conflicts of every depth, blocked admissions included."""
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import workload as W
    from test_gpu_batch import _compare_state
    from oracle.step import apply_warm_gpu
    B = 16
    rng = np.random.default_rng(seed)
    bases = [rng.integers(1, 1 << 62, size=int(rng.integers(8, 30)) * B + int(rng.integers(0, B)),
                          dtype=np.uint64) for _ in range(4)]
    R = 150
    prompts, pick = [], rng.integers(0, 4, R)
    for r in range(R):
        b = bases[pick[r]]
        cut = int(rng.integers(len(b) // 2, len(b) + 1))
        prompts.append(np.concatenate([b[:cut], rng.integers(1, 1 << 62, size=int(rng.integers(0, 40)),
                                                             dtype=np.uint64)]))
    lens = np.array([len(p) for p in prompts], np.int64)
    off = np.zeros(R + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    res = np.zeros(R, W.RES_DTYPE)
    res["prompt_len"] = lens
    res["upper"] = rng.integers(10, 300, R)
    res["alpha"] = np.where(rng.random(R) < 0.5, 0.0, 1 - 0.99)
    group = (rng.random(R) < 0.2).astype(np.int32)
    wf = (np.arange(R) // 3).astype(np.int32)
    role = rng.integers(0, 4, R).astype(np.int32)
    tr = W.Trace(torch.from_numpy(np.concatenate(prompts).view(np.int64)), off, res, group, wf, role)
    cl = W.make_cluster(10, 2, kv=6_000, l2=8_000, seed=seed, interleave=True, max_bg=1)
    ops = []
    for k, b in enumerate(bases):   # every chain into L3 via the completion sweep
        carrier = int(np.nonzero(pick == k)[0][0]) if (pick == k).any() else 0
        ops.append(("ins", k % cl.n_replicas, 1, carrier, int(lens[carrier]), 900 + k, 1, 0.1, 0))
        ops.append(("cmp", 900 + k, 0b10, 0.2))
    for r in range(0, R, 7):       # scattered L1/L2 prefixes
        ops.append(("ins", int(rng.integers(0, cl.n_replicas)), int(rng.integers(0, 2)), r,
                    int(rng.integers(0, lens[r] + 1)), int(wf[r]), int(role[r]),
                    float(rng.integers(0, 3)), 0))
    for w in range(int(wf.max()) + 1):
        ops.append(("reg", w, int(rng.integers(0, 16))))
    o, caches, l3, reg = _oracle(B, tr, cl, ops)
    ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, B)
    apply_warm_gpu(ctx, tr, ops)
    db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand)
    out = PB.alloc_out(ctx, db, dn)
    l3_hits = 0
    for s in range(3):
        now = 5.0 + s
        PB.step(ctx, db, dn, out, now)
        torch.cuda.synchronize()
        ctx.check_device_error()
        got = out.host()
        want = oracle_step(o, caches, l3, reg, tr, cl, SEQ_COMMIT, 0.05, now, True, True)
        assert [int(x) for x in got["decisions"]["target"][:R]] == [d[0] for d in want["decisions"]]
        assert np.array_equal(got["admitted"][:R], want["admitted"])
        assert np.array_equal(got["match3"][:R], want["match3"]), s
        _compare_state(o, caches, l3, ctx, cl)
        l3_hits += int((want["match3"][:, 2] > 0).sum())
    assert l3_hits > 0
