"""e2e breakdown (experiments): time the prompt-assembly e2e step's parts on one GPU with
CUDA events -- upload, assemble, device step, download."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    args = bench.parse()
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200.prompts import PromptPool
    dev = torch.device("cuda", 0)
    tr, cl = bench.build_workload(args, 0, 1, dev)
    ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, args.block)
    PB.bind_current_stream(ctx)
    bench.warm_l2(ctx, tr, cl, np.random.default_rng(0), n_workflows=bench.n_workflows_total(args, 1, tr))
    db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role, device=dev)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand, device=dev)
    out = PB.alloc_out(ctx, db, dn, device=dev)
    pool = PromptPool(tr, device=dev)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    h_res, h_grp, h_wf, h_role = pin(tr.res.view(np.int64).reshape(tr.R, 4)), pin(tr.group), pin(tr.wf), pin(tr.role)
    h_dec = torch.empty((tr.R, 3), dtype=torch.int64).pin_memory()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    acc = np.zeros(4)
    for it in range(13):
        ev[0].record()
        pool.upload()
        db.res.copy_(h_res, non_blocking=True); db.group.copy_(h_grp, non_blocking=True)
        db.wf.copy_(h_wf, non_blocking=True); db.role.copy_(h_role, non_blocking=True)
        ev[1].record()
        PB.bind_current_stream(ctx)
        pool.assemble(ctx, db.tok_off, db.tokens)
        bench._lib_check(ctx, db)
        ev[2].record()
        PB.step(ctx, db, dn, out, 1.0 + it)
        ev[3].record()
        h_dec.copy_(out.decisions[:tr.R], non_blocking=True)
        ev[4].record()
        torch.cuda.synchronize()
        if it >= 3:
            acc += [ev[k].elapsed_time(ev[k + 1]) for k in range(4)]
    acc /= 10
    print("upload %.3f ms  assemble %.3f ms  step %.3f ms  download %.3f ms  (h2d %d B, fresh %d tok)"
          % (*acc, pool.h2d_bytes, pool.fresh_tokens))


if __name__ == "__main__":
    main()
