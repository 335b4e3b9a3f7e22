"""GPU parity of device prompt assembly (csrc/k_prompt.cu): prompts gathered
from the resident pool + fresh tokens equal the workload's materialized prompts token for
token, and the step run on them equals the step on uploaded tokens."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["deep_research", "bursty", "coding", "long_context"])
def test_assembled_prompts_equal_materialized(kind):
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import workload as W
    from paper_2604_25899_b200.prompts import PromptPool
    tr = {"deep_research": lambda: W.deep_research(n_workflows=40, seed=3, device="cpu"),
          "bursty": lambda: W.bursty(n_requests=300, seed=3, device="cpu", mean_len=800),
          "coding": lambda: W.coding_assistant(n_workflows=6, seed=3, device="cpu"),
          "long_context": lambda: W.long_context(n_requests=6, seed=3, device="cpu")}[kind]()
    ctx = Context(1, 1000, 1000, 16)
    ctx.set_stream(None)
    pool = PromptPool(tr, device="cuda")
    tok_off = torch.empty(tr.R + 1, dtype=torch.int64, device="cuda")
    toks = torch.empty(max(tr.n_tokens, 1), dtype=torch.int64, device="cuda")
    pool.upload()
    pool.assemble(ctx, tok_off, toks)
    torch.cuda.synchronize()
    assert np.array_equal(tok_off.cpu().numpy(), tr.tok_off)
    assert torch.equal(toks[:tr.n_tokens].cpu(), tr.tokens.cpu())
    assert pool.h2d_bytes < tr.n_tokens * 8


N_STEPS = 5  # > 3 staging sets: the staging sets are reused


def test_pipelined_steps_equal_serial_steps():
    """PipelinedSteps (upload, assembly and K1 of later steps overlapped with step k) gives
    the same decisions, admissions and cache state as running the steps one after another
    on uploaded tokens."""
    from batch_oracle import apply_warm_gpu, warm_ops
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import workload as W
    from paper_2604_25899_b200.prompts import PipelinedSteps
    tr = W.deep_research(n_workflows=30, seed=4, device="cpu")
    cl = W.make_cluster(6, 2, kv=30_000, l2=30_000, seed=2)
    ops = warm_ops(tr, cl, 1)
    ctxs, results = [], []
    for pipelined in (False, True):
        ctx = Context(6, cl.kv_capacity, cl.l2_capacity, 16)
        apply_warm_gpu(ctx, tr, ops)
        db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role)
        dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off,
                             cl.cand)
        out = PB.alloc_out(ctx, db, dn)
        got = []
        if not pipelined:
            for k in range(N_STEPS):
                PB.step(ctx, db, dn, out, 5.0 + k)
                got.append(out.host())
        else:
            def run_step(b, k, after_gather):
                # hash offsets and K1 already ran on the pipeline's prep stream
                PB.staged_matrix(ctx, b, dn, out)
                after_gather()
                PB.route_batch(ctx, b, dn, out, PB.SEQ_COMMIT)
                PB.admit_batch(ctx, b, out, 5.0 + k, True)
                PB.release_batch(ctx, b, out)
                return out.decisions[:tr.R], out.admitted[:tr.R], out.match3[:tr.R]
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
            meta = (pin(tr.res.view(np.int64).reshape(tr.R, 4)), pin(tr.group), pin(tr.wf),
                    pin(tr.role))
            pipe = PipelinedSteps(ctx, tr, db, "cuda", run_step, meta,
                                  (out.decisions[:tr.R], out.admitted[:tr.R], out.match3[:tr.R]))
            pipe.run(N_STEPS)
            got = [None] * (N_STEPS - 1)
            got.append({"decisions": pipe.results[0][0].numpy(),
                        "admitted": pipe.results[0][1].numpy(),
                        "match3": pipe.results[0][2].numpy()})
        torch.cuda.synchronize()
        ctxs.append(ctx)
        results.append(got)
    serial, piped = results
    # the last step ran on batch set 0 (even steps): compare its outputs, then the caches
    assert np.array_equal(serial[-1]["decisions"].view(np.int64).reshape(-1, 3)[:tr.R],
                          piped[-1]["decisions"].reshape(-1, 3))
    assert np.array_equal(serial[-1]["admitted"][:tr.R], piped[-1]["admitted"])
    assert np.array_equal(serial[-1]["match3"][:tr.R], piped[-1]["match3"])
    for n in range(6):
        for t in (0, 1):
            assert ctxs[0].dump(n, t).tobytes() == ctxs[1].dump(n, t).tobytes(), (n, t)
    assert ctxs[0].dump(0, 2).tobytes() == ctxs[1].dump(0, 2).tobytes()


def _check_assemble_hash(pool, tr, B):
    """pyg_assemble_hash_dev == materialized prompts + the oracle's chain hashes."""
    from oracle.py_oracle import Restated
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    ctx = Context(0, [], [], B)
    ctx.set_stream(None)
    R = tr.R
    nb = (np.diff(tr.tok_off) + B - 1) // B
    b = PB.DeviceBatch(R, torch.full((max(tr.n_tokens, 1),), -1, dtype=torch.int64, device="cuda"),
                       torch.empty(R + 1, dtype=torch.int64, device="cuda"),
                       torch.empty(R + 1, dtype=torch.int64, device="cuda"),
                       torch.empty(max(int(nb.sum()), 1), dtype=torch.int64, device="cuda"),
                       None, None, None, None, int(nb.sum()), tr.n_tokens)
    pool.upload()
    pool.assemble_hash(ctx, b)
    torch.cuda.synchronize()
    ctx.check_device_error()
    assert np.array_equal(b.tok_off.cpu().numpy(), tr.tok_off)
    toks = tr.tokens_np()
    assert np.array_equal(b.tokens[:tr.n_tokens].cpu().numpy().view(np.uint64), toks)
    hoff = b.hash_off.cpu().numpy()
    assert hoff[0] == 0 and np.array_equal(np.diff(hoff), nb)
    got = b.hashes.cpu().numpy().view(np.uint64)
    o = Restated(B)
    for r in range(R):
        want = o.chain_hashes(toks[tr.tok_off[r]:tr.tok_off[r + 1]])
        assert np.array_equal(got[hoff[r]:hoff[r + 1]], want), r


@pytest.mark.parametrize("kind", ["deep_research", "bursty", "coding", "long_context"])
def test_assemble_hash_equals_materialized(kind):
    """K1 fused with the gather on every workload shape."""
    from paper_2604_25899_b200 import workload as W
    from paper_2604_25899_b200.prompts import PromptPool
    tr = {"deep_research": lambda: W.deep_research(n_workflows=40, seed=5, device="cpu"),
          "bursty": lambda: W.bursty(n_requests=300, seed=5, device="cpu", mean_len=800),
          "coding": lambda: W.coding_assistant(n_workflows=6, seed=5, device="cpu"),
          "long_context": lambda: W.long_context(n_requests=6, seed=5, device="cpu")}[kind]()
    _check_assemble_hash(PromptPool(tr, device="cuda"), tr, 16)


class _SynthPool:
    """Random segment layouts over a random pool: empty segments, segments shorter than a
    16-token chunk, many segments per chunk, requests with no segments."""

    def __init__(self, seed):
        rng = np.random.default_rng(seed)
        P = 50_000
        self.pool = torch.from_numpy(rng.integers(0, 1 << 62, P, dtype=np.int64)).cuda()
        R = 700
        nseg = rng.integers(0, 14, R)
        nseg[:5] = 0
        segs, lens = [], np.zeros(R, np.int64)
        for r in range(R):
            for _ in range(nseg[r]):
                kind = rng.integers(0, 4)
                L = [0, int(rng.integers(1, 16)), int(rng.integers(16, 200)),
                     int(rng.integers(200, 3000))][kind]
                src = int(rng.integers(0, P - L + 1))
                segs.append((src, L))
                lens[r] += L
        seg_off = np.zeros(R + 1, np.int64)
        np.cumsum(nseg, out=seg_off[1:])
        self.R = R
        self.d_seg_off = torch.from_numpy(seg_off).cuda()
        self.d_segs = torch.tensor(segs if segs else [(0, 0)], dtype=torch.int64).cuda()
        pool_h = self.pool.cpu().numpy().view(np.uint64)
        toks = [pool_h[s:s + L] for s, L in segs]
        self.tokens = np.concatenate(toks) if toks else np.zeros(0, np.uint64)
        self.tok_off = np.zeros(R + 1, np.int64)
        np.cumsum(lens, out=self.tok_off[1:])
        self.n_tokens = int(self.tok_off[-1])

    def upload(self):
        pass

    def tokens_np(self):
        return self.tokens

    def assemble_hash(self, ctx, b):
        from paper_2604_25899_b200 import _lib
        from paper_2604_25899_b200.prompts import _p
        _lib.check(_lib._lib.pyg_assemble_hash_dev(ctx.h, self.R, _p(self.d_seg_off),
                                                   _p(self.d_segs), int(self.d_segs.shape[0]),
                                                   _p(self.pool), self.n_tokens, _p(b.tok_off),
                                                   _p(b.tokens), _p(b.hash_off), _p(b.hashes)))


@pytest.mark.parametrize("B", [1, 5, 16, 64])
def test_assemble_hash_random_segments(B):
    sp = _SynthPool(B)
    _check_assemble_hash(sp, sp, B)
