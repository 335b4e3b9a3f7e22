"""GPU parity of K6 (csrc/k_nextuse.cu): expected_distance_to / future_roles for every
located history of the reference golden set, bit for bit (the BASELINE.json bar is 1e-6
relative; the kernel uses explicitly rounded FP64 so it is exact); per-block predicted next
use and the FutureRegistry update derived from it."""
import gzip
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import path_oracle as P

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "nextuse_golden.json.gz")


def _gold():
    with gzip.open(GOLD, "rt") as f:
        return json.load(f)


def _concat(cases):
    """All expressions in one node table (ids offset), cursors re-based."""
    keys = ["kind", "role", "min", "max", "p_continue", "p", "child", "ch_begin", "ch_end"]
    tab = {k: [] for k in keys}
    tab["ch_list"] = []
    frames, want = [], []
    for c in cases:
        t = c["table"]
        nb, cb = len(tab["kind"]), len(tab["ch_list"])
        for k in keys:
            v = t[k]
            if k == "child":
                v = [x + nb if x >= 0 else -1 for x in v]
            elif k in ("ch_begin", "ch_end"):
                v = [x + cb for x in v]
            tab[k].extend(v)
        tab["ch_list"].extend(x + nb for x in t["ch_list"])
        for q in c["queries"]:
            frames.append([(n + nb, p) for n, p in q["frames"]])
            want.append(q)
    return tab, frames, want


def test_next_use_matches_reference_golden():
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200.nextuse import PathTable, next_use
    g = _gold()
    tab, frames, want = _concat(g["cases"])
    ctx = Context(1, 1000, 1000, 16)
    t = PathTable(tab)
    ctx.set_stream(None)
    dist, fut = next_use(ctx, t, frames, g["n_roles"])
    torch.cuda.synchronize()
    d = dist.cpu().numpy()
    f = fut.cpu().numpy().view(np.uint64)
    for i, q in enumerate(want):
        assert int(f[i]) == q["future_mask"], (i, q["history"])
        for role in range(g["n_roles"]):
            w = q["distance"][role]
            if w is None:
                assert math.isnan(d[i, role]), (i, role)
            else:
                assert float(d[i, role]).hex() == w, (i, role, d[i, role], float.fromhex(w))


def test_block_next_use_and_registry_from_cursors():
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200.nextuse import (PathTable, block_next_use, next_use,
                                               registry_from_cursors)
    g = _gold()
    case = g["cases"][0]  # the config-2 deep-research shape
    nodes = P.from_table(case["table"])
    qs = case["queries"][:8]
    frames = [[tuple(x) for x in q["frames"]] for q in qs]
    ctx = Context(1, 100_000, 100_000, 16)
    ctx.set_stream(None)
    dist, fut = next_use(ctx, PathTable(case["table"]), frames, g["n_roles"])
    # blocks of workflows 0..7 (cursor i) and 8 (no cursor), every role
    rng = np.random.default_rng(1)
    blocks = []
    for k in range(40):
        w, r = int(rng.integers(0, 9)), int(rng.integers(0, g["n_roles"]))
        toks = rng.integers(1, 1 << 40, 16, dtype=np.uint64)
        ctx.insert_chain(0, 0, toks, 16, w, r, 1.0, 0)
        blocks.append((w, r))
    wf_cursor = torch.tensor(list(range(8)) + [-1], dtype=torch.int32, device="cuda")
    got = block_next_use(ctx, 0, 0, wf_cursor, dist).cpu().numpy()
    dump = ctx.dump(0, 0)
    assert len(got) == len(dump)
    for k, b in enumerate(dump):
        w, r = int(b["wf"]), int(b["role"])
        want = P.expected_distance_to(nodes, frames[w], r) if w < 8 else None
        if want is None:
            assert math.isnan(got[k])
        else:
            assert got[k] == want
    # FutureRegistry at issue = future_roles | current role (engine.cpp:605-609): eviction of
    # dead-lineage blocks first follows from it
    wf = torch.arange(8, dtype=torch.int32, device="cuda")
    cur_role = torch.tensor([q["history"][-1] for q in qs], dtype=torch.int32, device="cuda")
    registry_from_cursors(ctx, wf, wf.clone(), fut, cur_role, max_wf=8)
    torch.cuda.synchronize()
    from oracle.py_oracle import Restated
    o = Restated(16)
    c = o.new_cache(100_000, 100_000)
    reg = o.new_registry()
    for i, q in enumerate(qs):
        o.reg_update(reg, i, int(q["future_mask"]) | (1 << q["history"][-1]))
    rng = np.random.default_rng(1)
    for k in range(40):
        w, r = int(rng.integers(0, 9)), int(rng.integers(0, g["n_roles"]))
        toks = rng.integers(1, 1 << 40, 16, dtype=np.uint64)
        o.insert_chain(c, 0, toks, 16, w, r, 1.0, 0)
    freed_gpu = ctx.evict_for_space(0, 0, 100_000, True)
    freed_ref = o.evict_ids(c, 0, 100_000, reg, True)
    assert freed_gpu[0] == freed_ref[0] and freed_gpu[2] == freed_ref[2]
    assert list(freed_gpu[1]) == list(freed_ref[1]) and len(freed_gpu[1]) > 0
