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
        from paper_2604_25899_b200.shard import (ShardPlan, a2a, allgather_cat, allgather_var,
                                                 csr_offsets, dispatch_plan, local_placed,
                                                 pack_payload, unpack_payload)
        B = 16
        rng = np.random.default_rng(0)  # same global data on every rank
        reps = [3, 5, 2][:world]
        reqs = [7, 0, 9][:world] if world == 3 else [11, 6]
        R = sum(reqs)
        n_global = sum(reps)
        lens = rng.integers(0, 70, R)
        toks = [rng.integers(1, 1 << 40, int(n)) for n in lens]
        target = np.where(rng.random(R) < 0.6, rng.integers(0, n_global, R), -1)
        plan = ShardPlan(reps, reqs, rank, B)
        lo, hi = plan.req_base, plan.req_base + plan.R_local
        # payload round trip
        res = torch.from_numpy(rng.integers(0, 1 << 40, (R, 4)))
        grp = torch.from_numpy(rng.integers(0, 5, R).astype(np.int32))
        stg = torch.from_numpy(rng.integers(0, 9999, (R, 3)).astype(np.int32))
        L = torch.from_numpy(lens.astype(np.int64))
        pay = pack_payload(res[lo:hi], grp[lo:hi], grp[lo:hi] + 1, grp[lo:hi] + 2, L[lo:hi],
                           stg[lo:hi])
        g = unpack_payload(allgather_var(pay, reqs))
        assert torch.equal(g[0], res) and torch.equal(g[1], grp) and torch.equal(g[4], L)
        assert torch.equal(g[2], grp + 1) and torch.equal(g[3], grp + 2)
        assert torch.equal(g[5], stg)
        # variable all-gather
        mine = torch.arange(rank + 1, dtype=torch.int64) + 100 * rank
        allv = allgather_var(mine, [k + 1 for k in range(world)])
        assert allv.tolist() == [100 * k + i for k in range(world) for i in range(k + 1)]
        # dispatch
        tgt = torch.from_numpy(target.astype(np.int32))
        dp = dispatch_plan(plan, tgt, L)
        my_t = [torch.from_numpy(t.astype(np.int64)) for t in toks[lo:hi]]
        ltok = torch.cat(my_t) if my_t else torch.zeros(0, dtype=torch.int64)
        loff = csr_offsets(L[lo:hi])
        send = _gather_csr(ltok, loff, dp.send_idx)
        assert send.numel() == sum(dp.send_tok)
        recv = a2a(send, dp.send_tok, dp.recv_tok)
        owner = np.searchsorted(plan.rep_off[1:], target, side="right")
        want_g = [r for r in range(R) if target[r] >= 0 and owner[r] == rank]
        assert dp.recv_gidx.tolist() == want_g
        want = np.concatenate([toks[r] for r in want_g]) if want_g else np.zeros(0, np.int64)
        assert recv.tolist() == want.tolist()
        # local placed lists: global placed CSR (placement order = ascending index here)
        order = np.argsort(np.where(target >= 0, target, n_global), kind="stable")
        cnt = np.bincount(target[target >= 0], minlength=n_global)
        poff = torch.from_numpy(np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32))
        placed = torch.from_numpy(order[:int(cnt.sum())].astype(np.int32))
        p_off, p_loc = local_placed(plan, poff, placed, dp.recv_gidx)
        for n in range(plan.n_local):
            gl = [want_g[int(i)] for i in p_loc[int(p_off[n]):int(p_off[n + 1])]]
            assert gl == [r for r in range(R) if target[r] == plan.rep_base + n]
        # results back to origins
        back = torch.tensor([[r * 10, r] for r in dp.recv_gidx.tolist()],
                            dtype=torch.int64).reshape(-1, 2)
        ret = a2a(back, dp.recv_counts, dp.send_counts)
        got = {int(lo + i): int(v) for i, v in zip(dp.send_idx.tolist(), ret[:, 0].tolist())}
        for r in range(lo, hi):
            if target[r] >= 0:
                assert got[r] == r * 10
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
