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
