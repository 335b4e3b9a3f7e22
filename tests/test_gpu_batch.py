"""GPU parity of the batched step (K1 hash, K2 staged matrix, K3 route in both
modes, K4/K5 admission + release) against the oracle composition in
tests/batch_oracle.py, over several consecutive steps on an evolving cluster."""
import numpy as np
import pytest
import torch

from batch_oracle import (SEQ_COMMIT, SNAPSHOT, apply_warm_gpu, apply_warm_oracle, oracle_step,
                          warm_ops)
from oracle.py_oracle import Restated

pytestmark = pytest.mark.gpu


def _setup(trace, cl, B, seed):
    from paper_2604_25899_b200 import Context
    o = Restated(B)
    caches = [o.new_cache(int(cl.kv_capacity[n]), int(cl.l2_capacity[n]))
              for n in range(cl.n_replicas)]
    l3, reg = o.new_l3(), o.new_registry()
    ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, B)
    ops = warm_ops(trace, cl, seed)
    apply_warm_oracle(o, caches, l3, reg, trace, ops)
    apply_warm_gpu(ctx, trace, ops)
    return o, caches, l3, reg, ctx


def _compare_state(o, caches, l3, ctx, cl):
    for n in range(cl.n_replicas):
        for tier in (0, 1):
            g = ctx.dump(n, tier)
            w = o.dump(caches[n], None, tier)
            assert g.tobytes() == w.tobytes(), f"replica {n} tier {tier} differs"
    assert ctx.dump(0, 2).tobytes() == o.dump(caches[0], l3, 2).tobytes(), "L3 differs"


def _run(trace, cl, B, mode, steps, seed=0, spec=True):
    from paper_2604_25899_b200 import batch as PB
    o, caches, l3, reg, ctx = _setup(trace, cl, B, seed)
    db = PB.upload_batch(ctx, trace.tokens_np(), trace.tok_off, trace.res, trace.group, trace.wf,
                         trace.role)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand)
    out = PB.alloc_out(ctx, db, dn)
    total_placed = 0
    for s in range(steps):
        now = 10.0 + s
        PB.step(ctx, db, dn, out, now, mode=mode, speculative=spec, release=True)
        torch.cuda.synchronize()
        ctx.check_device_error()
        got = out.host()
        want = oracle_step(o, caches, l3, reg, trace, cl, mode, 0.05, now, spec, True)
        # hashes
        hs = db.hashes.cpu().numpy().view(np.uint64)
        for r in range(0, trace.R, max(1, trace.R // 50)):
            hw = o.chain_hashes(trace.prompt(r))
            a = int(db.hash_off[r].item())
            assert np.array_equal(hs[a:a + len(hw)], hw)
        assert np.array_equal(got["staged"][:trace.R], want["staged"])
        d = got["decisions"][:trace.R]
        for r in range(trace.R):
            wt = want["decisions"][r]
            assert (int(d["target"][r]), int(d["tiebreak"][r]), int(d["headroom"][r])) == wt[:3], r
            assert d["oom_bound"][r].tobytes() == np.float64(wt[3]).tobytes(), r
        po = got["placed_off"]
        for n in range(cl.n_replicas):
            assert got["placed"][po[n]:po[n + 1]].tolist() == want["placed"][n]
        assert np.array_equal(got["admitted"][:trace.R], want["admitted"])
        assert np.array_equal(got["match3"][:trace.R], want["match3"])
        _compare_state(o, caches, l3, ctx, cl)
        total_placed += int(sum(len(p) for p in want["placed"]))
    return total_placed


@pytest.mark.parametrize("B", [16, 64])
def test_batch_seq_commit_deep_research(B):
    from paper_2604_25899_b200 import workload as W
    tr = W.deep_research(n_workflows=24, seed=5, device="cpu")
    cl = W.make_cluster(8, 2, kv=24_000, l2=30_000, seed=1)
    placed = _run(tr, cl, B, SEQ_COMMIT, steps=3)
    assert placed > 10  # admissions and evictions were exercised


def test_batch_snapshot_small():
    from paper_2604_25899_b200 import workload as W
    tr = W.deep_research(n_workflows=4, seed=7, device="cpu")
    cl = W.make_cluster(6, 2, kv=400_000, l2=30_000, seed=2)
    _run(tr, cl, 16, SNAPSHOT, steps=2)


def test_batch_mixed_alphas_and_lru_only():
    from paper_2604_25899_b200 import workload as W
    tr = W.deep_research(n_workflows=16, seed=9, device="cpu")
    rng = np.random.default_rng(0)
    k = rng.random(tr.R)
    tr.res["alpha"] = np.where(k < 0.2, 0.02, np.where(k < 0.3, 0.0, tr.res["alpha"]))
    tr.res["alpha"][np.nonzero(k > 0.95)[0]] = -0.0
    cl = W.make_cluster(8, 2, kv=20_000, l2=20_000, seed=3)
    _run(tr, cl, 16, SEQ_COMMIT, steps=2, spec=False)


def test_batch_coding_assistant_chat_accumulate():
    from paper_2604_25899_b200 import workload as W
    tr = W.coding_assistant(n_workflows=12, seed=2, device="cpu")
    cl = W.make_cluster(4, 1, kv=40_000, l2=40_000, seed=4)
    _run(tr, cl, 16, SEQ_COMMIT, steps=3)


@pytest.mark.parametrize("B", [1, 5, 16, 32, 48, 64])
def test_hash_batch_all_lengths(B):
    """K1 over ragged batches: every length 0..300 and some long ones, odd/even starts."""
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    rng = np.random.default_rng(B)
    lens = np.concatenate([np.arange(0, 301), rng.integers(1000, 5000, 40)])
    rng.shuffle(lens)
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = rng.integers(0, 1 << 63, size=int(off[-1]), dtype=np.uint64) * np.uint64(2)
    ctx = Context(1, 1000, 1000, B)
    z = np.zeros(len(lens), np.int32)
    res = np.zeros(len(lens), PB.RES_DTYPE)
    db = PB.upload_batch(ctx, toks, off, res, z, z, z)
    PB.bind_current_stream(ctx)
    PB.hash_batch(ctx, db)
    torch.cuda.synchronize()
    got = db.hashes.cpu().numpy().view(np.uint64)
    hoff = db.hash_off.cpu().numpy()
    o = Restated(B)
    for r in range(len(lens)):
        want = o.chain_hashes(toks[off[r]:off[r + 1]])
        assert np.array_equal(got[hoff[r]:hoff[r + 1]], want), (r, lens[r])


@pytest.mark.parametrize("B", [16, 64])
def test_hash_batch_long_prompts_isolated(B):
    """K1's isolated long-task path: more than one task of prompts >= 8192 tokens (they run
    one warp per scheduler on their own SMs) mixed with a persistent pool of short ones."""
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    rng = np.random.default_rng(100 + B)
    lens = np.concatenate([rng.integers(8192, 12000, 70), [8192, 8191, 16384],
                           rng.integers(0, 3000, 2400)])
    rng.shuffle(lens)
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = rng.integers(0, 1 << 63, size=int(off[-1]), dtype=np.uint64)
    ctx = Context(1, 1000, 1000, B)
    z = np.zeros(len(lens), np.int32)
    res = np.zeros(len(lens), PB.RES_DTYPE)
    db = PB.upload_batch(ctx, toks, off, res, z, z, z)
    PB.bind_current_stream(ctx)
    PB.hash_batch(ctx, db)
    torch.cuda.synchronize()
    got = db.hashes.cpu().numpy().view(np.uint64)
    hoff = db.hash_off.cpu().numpy()
    o = Restated(B)
    for r in range(len(lens)):
        want = o.chain_hashes(toks[off[r]:off[r + 1]])
        assert np.array_equal(got[hoff[r]:hoff[r + 1]], want), (r, lens[r])


@pytest.mark.parametrize("B", [16, 64])
@pytest.mark.parametrize("split_min", [-1, 100])
def test_hash_batch_prefix_memo(B, split_min):
    """K1's prefix memo: requests sharing leading tokens with the leader of their first-16-token
    content start their chains after the leading chunks equal to the leader's (memo states;
    k_memo_emit writes those boundary hashes).  Shared lengths around every chunk / block /
    memo edge (0, 15..17, 31..33, 63..65, 2047..2049, whole prefixes), identical duplicates,
    one-bit mismatches, leaders shorter than followers, first chunks shared by 1-2 requests
    only (no memo row), prompts under 16 tokens; with the adaptive threshold and with most
    requests as split tasks (which start at the memo state too); the same batch memo off."""
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    rng = np.random.default_rng(900 + B + split_min)
    pre = [rng.integers(0, 1 << 63, size=n, dtype=np.uint64) for n in (40, 500, 2047, 2048,
                                                                      2049, 5000)]
    seqs = []
    for i in range(1600):
        p = pre[int(rng.integers(0, len(pre)))]
        k = int(rng.choice([0, 15, 16, 17, 31, 32, 33, 63, 64, 65, 2047, 2048, 2049, len(p),
                            len(p), int(rng.integers(0, len(p) + 1))]))
        k = min(k, len(p))
        tail = rng.integers(0, 1 << 63, size=int(rng.integers(0, 3000)), dtype=np.uint64)
        if i % 7 == 0 and k < len(p) and len(tail):
            tail[0] = p[k] ^ np.uint64(1)  # differs only in the low bit
        if i % 11 == 0 and k >= 16:
            tail = tail[:0]  # exactly a prefix of the shared content
        seqs.append(np.concatenate([p[:k], tail]))
        if i % 13 == 0:
            seqs.append(seqs[-1].copy())  # identical duplicate
    seqs += [rng.integers(0, 1 << 63, size=n, dtype=np.uint64) for n in range(0, 20)]
    order = rng.permutation(len(seqs))
    seqs = [seqs[j] for j in order]
    lens = np.array([len(x) for x in seqs])
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = np.concatenate(seqs).astype(np.uint64)
    o = Restated(B)
    want = [o.chain_hashes(toks[off[r]:off[r + 1]]) for r in range(len(lens))]
    for memo in (True, False):
        ctx = Context(1, 1000, 1000, B)
        ctx.set_hash_memo(memo)
        ctx.set_hash_split(split_min)
        z = np.zeros(len(lens), np.int32)
        res = np.zeros(len(lens), PB.RES_DTYPE)
        db = PB.upload_batch(ctx, toks, off, res, z, z, z)
        PB.bind_current_stream(ctx)
        for _ in range(2):  # the second call reuses the scratch of the first
            db.hashes.zero_()
            PB.hash_batch(ctx, db)
            torch.cuda.synchronize()
            ctx.check_device_error()
            got = db.hashes.cpu().numpy().view(np.uint64)
            hoff = db.hash_off.cpu().numpy()
            for r in range(len(lens)):
                assert np.array_equal(got[hoff[r]:hoff[r + 1]], want[r]), (memo, r, lens[r])


@pytest.mark.parametrize("grid", ["persistent", "tasks", "tasks1"])
@pytest.mark.parametrize("n_long", [40, 3000])
def test_hash_batch_grid_modes(grid, n_long):
    """K1's grid modes (persistent, one task per warp, one CTA per SM) on a sparse batch (few
    long one-lane chains: spread over the SMs, at most ceil(tasks / CTAs) warps per CTA) and
    a dense one, against the oracle."""
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    rng = np.random.default_rng(len(grid) * 31 + n_long)
    lens = np.concatenate([rng.integers(2000, 9000, n_long), rng.integers(0, 200, 60)])
    rng.shuffle(lens)
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = rng.integers(0, 1 << 63, size=int(off[-1]), dtype=np.uint64)
    ctx = Context(1, 1000, 1000, 16)
    ctx.set_hash_grid(grid)
    ctx.set_hash_split(0)  # one lane per request: the chains the spreading is for
    z = np.zeros(len(lens), np.int32)
    res = np.zeros(len(lens), PB.RES_DTYPE)
    db = PB.upload_batch(ctx, toks, off, res, z, z, z)
    PB.bind_current_stream(ctx)
    PB.hash_batch(ctx, db)
    torch.cuda.synchronize()
    got = db.hashes.cpu().numpy().view(np.uint64)
    hoff = db.hash_off.cpu().numpy()
    o = Restated(16)
    for r in range(len(lens)):
        assert np.array_equal(got[hoff[r]:hoff[r + 1]], o.chain_hashes(toks[off[r]:off[r + 1]])), \
            (grid, r, lens[r])


@pytest.mark.parametrize("B", [16, 32, 64, 5])
@pytest.mark.parametrize("split_min", [1, 100, 777])
def test_hash_batch_split_tasks(B, split_min):
    """K1 split tasks (one warp per prompt, low-byte decomposition of FNV-1a) with a low
    threshold so every length class goes through them: 1..1,100 tokens (partial segments,
    partial super-chunks, ragged block ends), super-chunk multiples, long prompts."""
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    rng = np.random.default_rng(7 * B + split_min)
    lens = np.concatenate([np.arange(0, 1100, 7), [511, 512, 513, 1024, 1025, 4096, 4097, 32768],
                           rng.integers(1, 20000, 60)])
    rng.shuffle(lens)
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = rng.integers(0, 1 << 63, size=int(off[-1]), dtype=np.uint64) * np.uint64(3)
    ctx = Context(1, 1000, 1000, B)
    ctx.set_hash_split(split_min)
    z = np.zeros(len(lens), np.int32)
    res = np.zeros(len(lens), PB.RES_DTYPE)
    db = PB.upload_batch(ctx, toks, off, res, z, z, z)
    PB.bind_current_stream(ctx)
    PB.hash_batch(ctx, db)
    torch.cuda.synchronize()
    got = db.hashes.cpu().numpy().view(np.uint64)
    hoff = db.hash_off.cpu().numpy()
    o = Restated(B)
    for r in range(len(lens)):
        want = o.chain_hashes(toks[off[r]:off[r + 1]])
        assert np.array_equal(got[hoff[r]:hoff[r + 1]], want), (r, lens[r])


def test_batch_config4_bursty_shape():
    """Config 4 shape: lognormal prompt lengths up to 32k, 4 models interleaved over the
    replicas, 10% unprofiled (alpha 0) reservations."""
    from paper_2604_25899_b200 import workload as W
    tr = W.bursty(n_requests=160, seed=4, device="cpu", mean_len=1500)
    cl = W.make_cluster(12, 4, kv=60_000, l2=60_000, seed=6, interleave=True)
    placed = _run(tr, cl, 16, SEQ_COMMIT, steps=2)
    assert placed > 10


def test_batch_config3_long_context_pressure():
    """Config 3 shape: 32,768-token prompts sharing a 28,672-token carried context,
    kv_capacity ~4 reservations, so capacity_holds binds alongside k_max."""
    from paper_2604_25899_b200 import workload as W
    tr = W.long_context(n_requests=24, seed=2, device="cpu")
    cl = W.make_cluster(6, 1, kv=141_000, l2=200_000, seed=7)
    placed = _run(tr, cl, 16, SEQ_COMMIT, steps=2)
    assert placed >= 6


@pytest.mark.parametrize("n_rep", [300, 1024])
def test_batch_config5_many_replicas(n_rep):
    """Config 5 sweep corner: up to 1024 replicas (16-word directory masks)."""
    from paper_2604_25899_b200 import workload as W
    tr = W.deep_research(n_workflows=6, seed=8, device="cpu")
    cl = W.make_cluster(n_rep, 2, kv=30_000, l2=30_000, seed=9, interleave=True, max_bg=1)
    _run(tr, cl, 16, SEQ_COMMIT, steps=1)


def test_batch_edge_cases_empty_and_no_candidates():
    """R = 0 through the device step and the host-buffer entry; a candidate group with no
    replicas (every request of it waits); zero-length prompts."""
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import workload as W
    cl = W.make_cluster(4, 2, kv=20_000, l2=20_000, seed=1)
    ctx = Context(4, cl.kv_capacity, cl.l2_capacity, 16)
    empty = np.zeros(0, PB.RES_DTYPE)
    z = np.zeros(0, np.int32)
    db = PB.upload_batch(ctx, np.zeros(1, np.uint64), np.zeros(1, np.int64), empty, z, z, z)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand)
    out = PB.alloc_out(ctx, db, dn)
    PB.step(ctx, db, dn, out, 1.0)
    torch.cuda.synchronize()
    ctx.check_device_error()
    # a group without candidates + empty prompts
    tr = W.deep_research(n_workflows=3, seed=2, device="cpu")
    grp = tr.group.copy()
    grp[::3] = 2                                      # group 2 has no replicas
    cand_off = np.concatenate([cl.cand_off, [cl.cand_off[-1]]]).astype(np.int32)
    lens = np.diff(tr.tok_off)
    lens[1::5] = 0
    off = np.zeros(tr.R + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = np.concatenate([tr.prompt(r)[:lens[r]] for r in range(tr.R)])
    res = tr.res.copy()
    res["prompt_len"] = lens
    o = Restated(16)
    caches = [o.new_cache(20_000, 20_000) for _ in range(4)]
    l3, reg = o.new_l3(), o.new_registry()
    db = PB.upload_batch(ctx, toks, off, res, grp, tr.wf, tr.role)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cand_off, cl.cand)
    out = PB.alloc_out(ctx, db, dn)
    PB.step(ctx, db, dn, out, 2.0)
    torch.cuda.synchronize()
    ctx.check_device_error()
    got = out.host()
    sub = W.Trace(torch.from_numpy(toks.view(np.int64)), off, res, grp, tr.wf, tr.role)

    class Cl:  # the cluster with the extra empty group
        pass
    c2 = Cl()
    c2.__dict__.update(cl.__dict__)
    c2.cand_off = cand_off
    want = oracle_step(o, caches, l3, reg, sub, c2, SEQ_COMMIT, 0.05, 2.0, True, True)
    d = got["decisions"][:tr.R]
    assert [int(x) for x in d["target"]] == [w[0] for w in want["decisions"]]
    assert all(int(d["target"][r]) == -1 for r in range(0, tr.R, 3))
    assert np.array_equal(got["admitted"][:tr.R], want["admitted"])
