"""One rank of the sharded steady-state parity check (tests/test_gpu_steady_shard.py launches
it through torchrun).  Every rank owns whole models' replicas and brings its own bursts
(paper_2604_25899_b200/steady_shard.py); rank 0 replays the same global bursts (the ranks'
bursts in rank order) through the unmodified reference on the whole cluster
(oracle/steady_ref.py) and every rank's share must match: each decision from its model's
owner, each admission / lookup from the owner that admitted it, every replica's L1/L2
tiers, and every rank's replica of the shared L3."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from oracle.py_oracle import DEC_DTYPE
    from oracle.steady_ref import RefSteady
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import steady as S
    from paper_2604_25899_b200 import workload as W
    from paper_2604_25899_b200.shard import allgather_cat
    from paper_2604_25899_b200.steady_shard import ShardedSteady

    dist.init_process_group("nccl", init_method="env://")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    B, R, K, n_models, per_model = 16, 300, 5, 4, 4
    kw = dict(mean_len=500, n_prefixes=24)
    cl = W.make_cluster(n_models * per_model, n_models, kv=24_000, l2=24_000, seed=5)
    warm = S.make_burst(10_000, 4 * R, 9, "cpu", "bursty", n_models, **kw)
    ops = S.warm_ops(warm, cl, l3_prefixes=16, l2_per_group=8, seed=5)
    off, placed = S.warm_fill_plan(warm, cl, fill_frac=0.97)
    per = cl.n_replicas // world
    lo, hi = rank * per, (rank + 1) * per
    ctx = Context(per, cl.kv_capacity[lo:hi], cl.l2_capacity[lo:hi], B, device=dev.index)
    PB.bind_current_stream(ctx)
    loc_off = (off[lo:hi + 1] - off[lo]).astype(np.int32)
    S.apply_warm_fill_gpu(ctx, warm, loc_off, placed[off[lo]:off[hi]], B, dev)
    S.apply_ops_gpu(ctx, warm, ops, rep_base=lo)
    subs = [[S.make_burst(k * world + g, R, 1, "cpu", "bursty", n_models, **kw)
             for g in range(world)] for k in range(K)]
    bursts = [S.upload_burst(subs[k][rank], B, dev, k * world + rank) for k in range(K)]
    sh = ShardedSteady(ctx, cl, rank, world, bursts, B, dev)
    sh.build_directory()
    ref = None
    if rank == 0:
        ref = RefSteady(B, cl, threads=4)
        ref.warm(warm, ops, off, placed)
    owner_of_group = {}
    for g in range(n_models):
        c = cl.cand[cl.cand_off[g]]
        owner_of_group[g] = int(c) // per
    bad = []
    for k in range(K):
        PB.bind_current_stream(ctx)
        PB.hash_batch(ctx, bursts[k].b)
        st = sh.step(k, 1.0 + k)
        torch.cuda.synchronize(dev)
        ctx.check_device_error()
        Rt = R * world
        dec = st.decisions[:Rt].contiguous()
        alld = allgather_cat(dec).cpu().numpy().view(DEC_DTYPE).reshape(world, Rt)
        # admitted / match3 per global request from the owner that admitted it
        n = int(st.recv_count.item())
        adm_g = torch.full((Rt,), -1, dtype=torch.int64, device=dev)
        m3_g = torch.full((Rt, 3), -1, dtype=torch.int64, device=dev)
        gi = st.recv_gidx[:n].long()
        adm_g[gi] = st.adm[:n].long()
        m3_g[gi] = st.m3[:n]
        dist.all_reduce(adm_g, op=dist.ReduceOp.MAX)
        dist.all_reduce(m3_g, op=dist.ReduceOp.MAX)
        if rank == 0:
            toks = np.concatenate([t.tokens_np() for t in subs[k]])
            lens = np.concatenate([np.diff(t.tok_off) for t in subs[k]])
            tok_off = np.zeros(Rt + 1, np.int64)
            np.cumsum(lens, out=tok_off[1:])
            cat = lambda f: np.concatenate([getattr(t, f) for t in subs[k]])  # noqa: E731
            hold = np.concatenate([S.hold_of(k * world + g, R, R) for g in range(world)])
            rw, rm = S.registry_pairs(cat("wf"), cat("role"))
            d, a, m3, _ = ref.step(k, toks, tok_off, cat("res"), cat("group"), cat("wf"),
                                   cat("role"), rw, rm, 1.0 + k, hold)
            grp = cat("group")
            got = np.array([alld[owner_of_group[int(grp[r])], r] for r in range(Rt)],
                           DEC_DTYPE)
            for f in ("target", "tiebreak", "headroom"):
                if not np.array_equal(got[f], d[f]):
                    bad.append((k, f, int(np.nonzero(got[f] != d[f])[0][0])))
            if got["oom_bound"].tobytes() != d["oom_bound"].tobytes():
                bad.append((k, "oom_bound"))
            ag = adm_g.cpu().numpy()
            pl = d["target"] >= 0
            if not np.array_equal(np.where(pl, ag, 0), a.astype(np.int64)):
                bad.append((k, "admitted"))
            if not np.array_equal(m3_g.cpu().numpy()[pl], m3[pl]):
                bad.append((k, "match3"))
    # tiers: every rank's replicas against the reference's
    dumps = [(lo + n, t, ctx.dump(n, t).tobytes()) for n in range(per) for t in (0, 1)]
    dumps.append((-1, 2, ctx.dump(0, 2).tobytes()))
    alld = [None] * world
    dist.all_gather_object(alld, dumps)
    if rank == 0:
        for part in alld:
            for n, t, b in part:
                want = ref.dump(0 if n < 0 else n, t).tobytes()
                if b != want:
                    bad.append(("tier", n, t))
        print("steady shard parity", "ok" if not bad else f"FAILED {bad[:10]}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
