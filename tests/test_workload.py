"""Synthetic traces use the reference's token conventions (CPU)."""
import numpy as np
import pytest
import torch

from paper_2604_25899_b200 import workload as W
from oracle.py_oracle import Reference, Restated, reference_available


def test_scalar_fnv_matches_oracle():
    o = Restated(16)
    for s in ["", "a", "sys_planner_17", "w12_s3_1"]:
        assert W.fnv1a_str(s) == o.fnv1a_str(s)
    for v in [0, 1, 255, 256, (1 << 64) - 1, 0x0123456789ABCDEF]:
        assert W.fnv1a_u64(v) == o.fnv1a_u64(v)


def test_vector_fnv_matches_scalar():
    rng = np.random.default_rng(0)
    v = rng.integers(-(1 << 63), (1 << 63) - 1, 1000, dtype=np.int64)
    h = rng.integers(-(1 << 63), (1 << 63) - 1, 1000, dtype=np.int64)
    out = W.fnv1a_u64_vec(torch.from_numpy(v), torch.from_numpy(h)).numpy().view(np.uint64)
    for a, b, c in zip(v.view(np.uint64), h.view(np.uint64), out):
        assert W.fnv1a_u64(int(a), int(b)) == int(c)


@pytest.mark.skipif(not reference_available(16), reason="oracle/_ref not built")
def test_response_token_matches_reference():
    ref = Reference(16)
    for rid in ["w0_s1_0", "w17_s3_2"]:
        for i in [0, 1, 99]:
            assert ref.response_token(rid, i) == W.fnv1a_u64(i, W.response_key(rid))


def test_deep_research_trace_shape():
    t = W.deep_research(n_workflows=20, seed=3, device="cpu")
    assert t.R == len(t.res) == len(t.group)
    assert np.all(np.diff(t.tok_off) == t.res["prompt_len"])
    # every researcher of one round shares sys + carried prefix with its siblings
    toks = t.tokens_np()
    r0 = np.nonzero(t.role == 1)[0][:2]
    a, b = t.prompt(r0[0]), t.prompt(r0[1])
    assert np.array_equal(a[:768], b[:768])
    # word tokens are fnv1a("sys_<role>_<i>")
    d = np.nonzero(t.role == 0)[0][0]
    assert int(t.prompt(d)[5]) == W.fnv1a_str("sys_decomposer_5")
    assert int(toks[t.tok_off[d] + 512]) == W.fnv1a_u64(0, W.task_key("w0"))


def test_other_configs_build():
    for t in [W.coding_assistant(5, device="cpu"), W.long_context(16, device="cpu"),
              W.bursty(64, device="cpu")]:
        assert t.R > 0 and t.n_tokens == int(np.diff(t.tok_off).sum())
