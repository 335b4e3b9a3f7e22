"""One rank of the sharded-step parity check (launched by tests/test_gpu_shard.py through
torchrun, or with WORLD_SIZE=1 in-process).  Every rank builds the same global trace and
cluster, owns a contiguous slice of replicas and requests, runs ShardedStep, and compares
its share of the result with the single-cluster oracle composition (oracle/step.py):
all route decisions, admissions/matches of its requests, the L1/L2 tiers of its
replicas and its replica of the shared L3."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.py_oracle import Restated  # noqa: E402
from oracle.step import SEQ_COMMIT, oracle_step  # noqa: E402


def split(n, world):
    base = [n // world + (1 if k < n % world else 0) for k in range(world)]
    return base


def l3_warm_ops(trace, rng, n=5):
    ops = []
    for r in rng.choice(trace.R, n, replace=False):
        ops.append((int(r), float(rng.integers(0, 4))))
    return ops


def run(rank, world, B=16, steps=3, n_wf=20, n_rep=8, n_models=2, interleave=True, seed=3):
    from oracle.step import warm_ops
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import workload as W
    from paper_2604_25899_b200.shard import ShardPlan, ShardedStep, decisions_host

    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    tr = W.deep_research(n_workflows=n_wf, seed=seed, device="cpu")
    cl = W.make_cluster(n_rep, n_models, kv=20_000, l2=30_000, seed=seed, interleave=interleave)
    reps = split(n_rep, world)
    reqs = split(tr.R, world)
    plan = ShardPlan(reps, reqs, rank, B)
    # oracle: the whole cluster
    o = Restated(B)
    caches = [o.new_cache(int(cl.kv_capacity[n]), int(cl.l2_capacity[n])) for n in range(n_rep)]
    l3, reg = o.new_l3(), o.new_registry()
    # this rank's GPU shard
    lo = plan.rep_base
    ctx = Context(plan.n_local, cl.kv_capacity[lo:lo + plan.n_local],
                  cl.l2_capacity[lo:lo + plan.n_local], B, device=dev.index)
    ops = [op for op in warm_ops(tr, cl, seed) if op[0] != "cmp"]
    for op in ops:
        if op[0] == "ins":
            _, n, tier, r, upto, wf, role, now, pin = op
            o.insert_chain(caches[n], tier, tr.prompt(r), upto, wf, role, now, pin)
            if lo <= n < lo + plan.n_local:
                ctx.insert_chain(n - lo, tier, tr.prompt(r), upto, wf, role, now, pin)
        elif op[0] == "reg":
            o.reg_update(reg, op[1], op[2])
            ctx.registry_update(op[1], op[2])
    rng = np.random.default_rng(seed + 1)
    for r, now in l3_warm_ops(tr, rng):  # the shared L3, replicated on every rank
        p = tr.prompt(r)
        hs = o.chain_hashes(p)
        upto = len(p) if rng.random() < 0.6 else int(rng.integers(1, len(p) + 1))
        for i, h in enumerate(hs):
            s, e = i * B, min((i + 1) * B, len(p))
            if e > upto:
                break
            o.put(caches[0], l3, 2, int(h), s, e, int(tr.wf[r]), int(tr.role[r]), now, 0)
            ctx.put(0, 2, int(h), s, e, int(tr.wf[r]), int(tr.role[r]), now, 0)
    sub = tr.subset(np.arange(plan.req_base, plan.req_base + plan.R_local))
    db = PB.upload_batch(ctx, sub.tokens_np(), sub.tok_off, sub.res, sub.group, sub.wf, sub.role,
                         device=dev)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand,
                         device=dev)
    st = ShardedStep(ctx, plan, db, dn, dev, cl.kv_capacity[lo:lo + plan.n_local], tr.n_tokens)
    st.build_directory()
    placed_total = 0
    for s in range(steps):
        now = 10.0 + s
        got = st.step(now)
        torch.cuda.synchronize()
        ctx.check_device_error()
        want = oracle_step(o, caches, l3, reg, tr, cl, SEQ_COMMIT, 0.05, now, True, True)
        d = decisions_host(got["decisions"])
        for r in range(tr.R):
            wt = want["decisions"][r]
            assert (int(d["target"][r]), int(d["tiebreak"][r]), int(d["headroom"][r])) == wt[:3], \
                (rank, s, r)
            assert d["oom_bound"][r].tobytes() == np.float64(wt[3]).tobytes(), (rank, s, r)
        a, b = plan.req_base, plan.req_base + plan.R_local
        assert np.array_equal(got["staged"].cpu().numpy(), want["staged"][a:b]), (rank, s)
        assert np.array_equal(got["admitted"].cpu().numpy(), want["admitted"][a:b]), (rank, s)
        assert np.array_equal(got["match3"].cpu().numpy(), want["match3"][a:b]), (rank, s)
        for n in range(plan.n_local):
            for tier in (0, 1):
                assert ctx.dump(n, tier).tobytes() == o.dump(caches[lo + n], None, tier).tobytes(), \
                    (rank, s, n, tier)
        assert ctx.dump(0, 2).tobytes() == o.dump(caches[0], l3, 2).tobytes(), (rank, s, "L3")
        placed_total += sum(len(p) for p in want["placed"])
    assert placed_total > 5
    return placed_total


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist.init_process_group("nccl", init_method="env://")
    cases = [dict(interleave=True), dict(interleave=False, n_rep=6, n_models=3, seed=5),
             dict(B=64, n_wf=12, seed=7)]
    for kw in cases:
        n = run(rank, world, **kw)
        if rank == 0:
            print(f"shard parity ok: world={world} {kw} placed={n}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
