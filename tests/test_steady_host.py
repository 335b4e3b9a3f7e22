"""Host-side logic of the steady-state step (CPU): model ownership of the sharded split,
placement holds, registry last-write pairs, the reference node-table composition, and the
world-2 gloo path that gathers a global burst's registry updates."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_25899_b200 import steady as S
from paper_2604_25899_b200 import workload as W


def test_owned_groups_split_by_model():
    from paper_2604_25899_b200.steady_shard import owned_groups
    cl = W.make_cluster(256, 8, seed=0)
    assert owned_groups(cl, 0, 256) == list(range(8))
    assert owned_groups(cl, 0, 128) == [0, 1, 2, 3]
    assert owned_groups(cl, 224, 256) == [7]
    with pytest.raises(ValueError):
        owned_groups(cl, 0, 48)  # model 1 = replicas 32..63 straddles
    cli = W.make_cluster(16, 4, seed=0, interleave=True)
    with pytest.raises(ValueError):
        owned_groups(cli, 0, 8)


def test_hold_of_global_ids():
    # burst k of R requests per burst: hold = 1 + parity of the global request id; a sharded
    # job's sub-burst k*W + g covers the same ids as the single-GPU burst numbering
    R = 6
    h = S.hold_of(3, R, R)
    assert h.tolist() == [1 + ((3 * R + r) & 1) for r in range(R)]
    W_ = 2
    cat = np.concatenate([S.hold_of(1 * W_ + g, R, R) for g in range(W_)])
    assert cat.tolist() == [1 + (((W_ + 0) * R + r) & 1) for r in range(W_ * R)]
    assert S.hold_of(0, 10, 4).tolist() == [1, 2, 1, 2]


def test_registry_pairs_last_write():
    wf = np.array([5, 7, 5, 9, 7, 5], np.int32)
    role = np.array([0, 1, 2, 3, 4, 5], np.int32)
    u, m = S.registry_pairs(wf, role)
    assert u.tolist() == [5, 7, 9]
    want = S.registry_mask(np.array([5, 4, 3], np.int32))  # last request of each workflow
    assert m.tolist() == want.tolist()


def test_ref_node_table_holds():
    from oracle.py_oracle import reference_available
    if not reference_available(16):
        pytest.skip("oracle/_ref not built")
    from oracle.steady_ref import RefSteady
    cl = W.make_cluster(4, 1, seed=1, max_bg=2)
    ref = RefSteady(16, cl)
    res = np.zeros(5, W.RES_DTYPE)
    res["prompt_len"] = np.arange(5) + 100
    tgt = np.array([0, 2, -1, 2, 3], np.int32)
    hold = np.array([2, 1, 2, 2, 1], np.uint8)
    ref.hist[0] = (None, None, tgt, np.ones(5, np.int32), res, hold)
    off, asg = ref.node_table(1)
    # base entries first, then burst 0's placements still held (hold 2) in placement order
    for n in range(4):
        base = cl.asg[cl.asg_off[n]:cl.asg_off[n + 1]]
        got = asg[off[n]:off[n + 1]]
        assert got[:len(base)].tobytes() == base.tobytes()
        extra = [int(x) for x in got["prompt_len"][len(base):]]
        want = [100 + r for r in range(5) if tgt[r] == n and hold[r] == 2]
        assert extra == want, n


def _gather_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_25899_b200.shard import allgather_cat
    R = 64
    subs = [S.make_burst(2 * world + g, R, 1, "cpu", "bursty", 8, mean_len=100, n_prefixes=8)
            for g in range(world)]
    mine = torch.from_numpy(subs[rank].wf)
    wf = allgather_cat(mine).numpy()
    role = allgather_cat(torch.from_numpy(subs[rank].role)).numpy()
    u, m = S.registry_pairs(wf, role)
    u0, m0 = S.registry_pairs(np.concatenate([t.wf for t in subs]),
                              np.concatenate([t.role for t in subs]))
    out[rank] = int(np.array_equal(u, u0) and np.array_equal(m, m0))
    dist.destroy_process_group()


def test_world2_registry_pairs_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_gather_worker, args=(2, port, out), nprocs=2, join=True)
    assert dict(out) == {0: 1, 1: 1}
