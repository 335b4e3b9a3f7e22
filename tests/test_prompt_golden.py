"""Device prompt assembly pinned to the reference: templates in the
reference's placeholder form over exchange histories, against vectors made by the
unmodified parse_prompt_template + assemble_prompt / assemble_resolvable_prefix
(tests/golden/make_prompt_golden.py): clamped and out-of-range slices, missing exchanges
(nullopt / prefix stop), literal words with mixed whitespace, malformed placeholders.
CPU: the host resolution (paper_2604_25899_b200/templates.py) gathered on the host.
GPU: the same resolution gathered by pyg_assemble_dev, a batch at a time."""
import gzip
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    with gzip.open(os.path.join(HERE, "golden", "prompt_golden.json.gz"), "rt") as f:
        return json.load(f)["cases"]


def _ex(c):
    return {k: (np.array(v[0], np.uint64), np.array(v[1], np.uint64)) for k, v in c["ex"].items()}


def test_host_resolution_matches_reference():
    from paper_2604_25899_b200 import templates as T
    n_ok = n_null = n_err = 0
    for c in _cases():
        pool = T.ExchangePool(_ex(c), device="cpu")
        for prefix in (0, 1):
            rc = c[f"rc{prefix}"]
            try:
                res = pool.resolve(c["text"], prefix=bool(prefix))
            except ValueError:
                assert rc == -1, c["text"]
                n_err += 1
                continue
            assert rc != -1, c["text"]
            if res is None:
                assert rc == 1 and not prefix
                n_null += 1
                continue
            segs, complete = res
            assert rc == 0
            assert complete == c[f"complete{prefix}"], c["text"]
            got = pool.gather_host(segs)
            assert got.tolist() == c[f"tok{prefix}"], c["text"]
            n_ok += 1
    assert n_ok > 200 and n_null > 20 and n_err > 20


@pytest.mark.gpu
def test_device_assembly_matches_reference():
    import torch
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import templates as T
    ctx = Context(0, [], [], 16)
    dev = torch.device("cuda", 0)
    for c in _cases():
        pool = T.ExchangePool(_ex(c), device=dev)
        batch, want = [], []
        for prefix in (0, 1):
            if c[f"rc{prefix}"] != 0:
                continue
            segs, _ = pool.resolve(c["text"], prefix=bool(prefix))
            batch.append(segs)
            want.append(c[f"tok{prefix}"])
        if not batch:
            continue
        tok_off, tokens = pool.assemble(ctx, batch)
        torch.cuda.synchronize()
        off = tok_off.cpu().numpy()
        toks = tokens.cpu().numpy().view(np.uint64)
        for k, w in enumerate(want):
            assert toks[off[k]:off[k + 1]].tolist() == w, c["text"]
