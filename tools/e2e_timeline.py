"""e2e pipeline timeline (experiments): runs bench.py's one-GPU e2e PipelinedSteps with a
CUDA event at every stage boundary and prints, per step, when each stage started/ended
(ms from the first upload) plus the host issue time per step."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    args = bench.parse()
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200.prompts import PipelinedSteps
    dev = torch.device("cuda", 0)
    S = torch.cuda.Stream(device=dev, priority=-1)
    torch.cuda.set_stream(S)
    tr, cl = bench.build_workload(args, 0, 1, dev)
    ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, args.block)
    PB.bind_current_stream(ctx)
    bench.warm_l2(ctx, tr, cl, np.random.default_rng(0),
                  n_workflows=bench.n_workflows_total(args, 1, tr))
    db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role,
                         device=dev)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand,
                         device=dev)
    out = PB.alloc_out(ctx, db, dn, device=dev)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    meta = (pin(tr.res.view(np.int64).reshape(tr.R, 4)), pin(tr.group), pin(tr.wf), pin(tr.role))

    def run_step(b, k, after_gather):
        PB.staged_matrix(ctx, b, dn, out)
        after_gather()
        PB.route_batch(ctx, b, dn, out, PB.SEQ_COMMIT)
        PB.admit_batch(ctx, b, out, 1.0 + k, True)
        PB.release_batch(ctx, b, out)
        return out.decisions[:tr.R], out.admitted[:tr.R], out.match3[:tr.R]

    pipe = PipelinedSteps(ctx, tr, db, dev, run_step, meta,
                          (out.decisions[:tr.R], out.admitted[:tr.R], out.match3[:tr.R]))
    pipe.run(3)
    pipe.marks = []
    n = 8
    t0 = time.perf_counter()
    pipe.run(n, first_index=3)
    wall = (time.perf_counter() - t0) * 1000
    marks = pipe.marks
    base = marks[0][2]
    rows = {}
    for name, k, e in marks:
        rows.setdefault(k, {})[name] = base.elapsed_time(e)
    print(f"wall {wall:.3f} ms for {n} steps = {wall / n:.3f} ms/step")
    names = ["upload0", "upload1", "prep0", "prep1", "step0", "step1", "d2h1"]
    print("step " + " ".join(f"{x:>8}" for x in names))
    for k in sorted(rows):
        print(f"{k:4d} " + " ".join(f"{rows[k].get(x, float('nan')):8.3f}" for x in names))


if __name__ == "__main__":
    main()
