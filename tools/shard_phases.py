"""Per-phase timing of the sharded step (run under torchrun): device time between phase
marks and host time, rank 0 prints a table."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    args = bench.parse()
    ws, rank, local = bench.dist_env()
    dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200.shard import ShardPlan, ShardedStep
    tr, cl = bench.build_workload(args, rank, ws, dev)
    n_loc, base = args.replicas, rank * args.replicas
    c = torch.tensor([tr.R], device=dev)
    allc = [torch.zeros_like(c) for _ in range(ws)]
    dist.all_gather(allc, c)
    plan = ShardPlan([n_loc] * ws, [int(x.item()) for x in allc], rank, args.block)
    ctx = Context(n_loc, cl.kv_capacity[base:base + n_loc], cl.l2_capacity[base:base + n_loc],
                  args.block, device=local)
    PB.bind_current_stream(ctx)
    bench.warm_l2(ctx, tr, cl, np.random.default_rng(rank), rep_base=base, n_local=n_loc,
                  n_workflows=ws * args.workflows)
    db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role, device=dev)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand, device=dev)
    st = ShardedStep(ctx, plan, db, dn, dev, cl.kv_capacity[base:base + n_loc])
    st.build_directory()
    for i in range(3):
        st.step(1.0 + i)
    torch.cuda.synchronize()
    dist.barrier()
    acc = {}
    for i in range(5):
        marks = []
        st.step(10.0 + i, marks=marks)
        torch.cuda.synchronize()
        for (n0, e0, h0), (n1, e1, h1) in zip(marks, marks[1:]):
            d = acc.setdefault(n1, [0.0, 0.0])
            d[0] += e0.elapsed_time(e1) / 5
            d[1] += (h1 - h0) * 1000 / 5
    if rank == 0:
        for k, (dv, hv) in acc.items():
            print(f"{k:16s} device {dv:8.3f} ms   host {hv:8.3f} ms")
        print("total device", sum(v[0] for v in acc.values()))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
