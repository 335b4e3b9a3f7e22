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


def test_pipelined_steps_equal_serial_steps():
    """PipelinedSteps (upload of step k+1 overlapped with step k) gives the same decisions,
    admissions and cache state as running the steps one after another on uploaded tokens."""
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
            for k in range(3):
                PB.step(ctx, db, dn, out, 5.0 + k)
                got.append(out.host())
        else:
            import ctypes as C
            from paper_2604_25899_b200 import _lib

            def run_step(b, k):
                _lib.check(_lib._lib.pyg_hash_offsets_dev(ctx.h, C.c_void_p(b.tok_off.data_ptr()),
                                                          b.R, C.c_void_p(b.hash_off.data_ptr()),
                                                          None))
                PB.hash_batch(ctx, b)
                PB.staged_matrix(ctx, b, dn, out)
                PB.route_batch(ctx, b, dn, out, PB.SEQ_COMMIT)
                PB.admit_batch(ctx, b, out, 5.0 + k, True)
                PB.release_batch(ctx, b, out)
                return out.decisions[:tr.R], out.admitted[:tr.R], out.match3[:tr.R]
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
            meta = (pin(tr.res.view(np.int64).reshape(tr.R, 4)), pin(tr.group), pin(tr.wf),
                    pin(tr.role))
            pipe = PipelinedSteps(ctx, tr, db, "cuda", run_step, meta,
                                  (out.decisions[:tr.R], out.admitted[:tr.R], out.match3[:tr.R]))
            pipe.run(3)
            got.append({"decisions": pipe.results[0][0].numpy(),
                        "admitted": pipe.results[0][1].numpy()})
            got.append({"decisions": pipe.results[0][0].numpy()})
            got.append({"decisions": pipe.results[0][0].numpy(),
                        "admitted": pipe.results[0][1].numpy(),
                        "match3": pipe.results[0][2].numpy()})
        torch.cuda.synchronize()
        ctxs.append(ctx)
        results.append(got)
    serial, piped = results
    # step 3 ran on input set 0 (steps 0 and 2 use set 0): compare the last step's outputs
    assert np.array_equal(serial[2]["decisions"].view(np.int64).reshape(-1, 3)[:tr.R],
                          piped[2]["decisions"].reshape(-1, 3))
    assert np.array_equal(serial[2]["admitted"][:tr.R], piped[2]["admitted"])
    assert np.array_equal(serial[2]["match3"][:tr.R], piped[2]["match3"])
    for n in range(6):
        for t in (0, 1):
            assert ctxs[0].dump(n, t).tobytes() == ctxs[1].dump(n, t).tobytes(), (n, t)
    assert ctxs[0].dump(0, 2).tobytes() == ctxs[1].dump(0, 2).tobytes()
