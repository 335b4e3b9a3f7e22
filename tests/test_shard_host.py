"""CPU (gloo, world_size 2 and 3) tests of the multi-GPU step's host logic
(paper_2604_25899_b200/shard.py): payload all-gather, the dispatch plan that sends
each placed request's tokens/hashes from its origin to its target's owner, the local
placed lists on the owner, and the return of results to the origins.  The device
kernel pyg_gather_csr_dev is replaced here by a torch gather (test-only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_csr(src, off, idx):
    parts = [src[int(off[i]):int(off[i + 1])] for i in idx.tolist()]
    return torch.cat(parts) if parts else src[:0]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2604_25899_b200.shard import (ShardPlan, allgather_cat, allgather_var,
                                                 exchange_windows)
        B = 16
        rng = np.random.default_rng(0)  # same global data on every rank
        reps = [3, 5, 2][:world]
        reqs = [7, 0, 9][:world] if world == 3 else [11, 6]
        R = sum(reqs)
        n_global = sum(reps)
        lens = rng.integers(0, 70, R)
        plan = ShardPlan(reps, reqs, rank, B)
        lo, hi = plan.req_base, plan.req_base + plan.R_local
        assert plan.n_global == n_global and plan.R_total == R
        # owner of every global replica id
        tg = torch.tensor([-1] + list(range(n_global)))
        want = [-1] + [int(np.searchsorted(plan.rep_off[1:], t, side="right"))
                       for t in range(n_global)]
        assert plan.owner(tg).tolist() == want
        # route rows through the variable all-gather (ranks hold different R; global order)
        rows = torch.from_numpy(rng.integers(-(1 << 31), 1 << 31, (R, 13)).astype(np.int32))
        g = allgather_var(rows[lo:hi].contiguous(), reqs)
        assert torch.equal(g, rows)
        assert lens.shape[0] == R
        mine = torch.arange(rank + 1, dtype=torch.int64) + 100 * rank
        allv = allgather_var(mine, [k + 1 for k in range(world)])
        assert allv.tolist() == [100 * k + i for k in range(world) for i in range(k + 1)]
        assert allgather_cat(torch.tensor([rank])).tolist() == list(range(world))
        # exchange windows: own pointers stay local, peers' come through import(handle, offset)
        local = [1000 * rank + f for f in range(11)]
        wins = exchange_windows(local, lambda p: (b"h%d" % p, p % 7),
                                lambda h, o: ("imported", h, o))
        for k in range(world):
            if k == rank:
                assert wins[k] == local
            else:
                assert wins[k] == [("imported", b"h%d" % (1000 * k + f), (1000 * k + f) % 7)
                                   for f in range(11)]
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_shard_host_logic_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=90) for _ in range(world)]
    for p in ps:
        p.join(60)
    for rank, msg in out:
        assert msg == "ok", f"rank {rank}:\n{msg}"
