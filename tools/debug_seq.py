import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2604_25899_b200 import Context, batch as PB
class A: pass
a = A(); a.workflows=10000; a.replicas=32; a.block=16; a.kv=100_000; a.l2=200_000
dev = torch.device("cuda", 0)
tr, cl = bench.build_workload(a, 0, dev)
ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, 16)
PB.bind_current_stream(ctx)
db = PB.upload_batch(ctx, tr.tokens_np(), tr.tok_off, tr.res, tr.group, tr.wf, tr.role)
dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand)
out = PB.alloc_out(ctx, db, dn)
PB.step(ctx, db, dn, out, 1.0)
torch.cuda.synchronize()
h = out.host()
tgt = h["decisions"]["target"][:tr.R]
pl = np.nonzero(tgt >= 0)[0]
print("placed", len(pl))
for g in range(2):
    p = pl[tr.group[pl] == g]
    ch = np.unique(p // 128)
    print("group", g, "placements", len(p), "distinct chunks", len(ch), "last placement idx", p.max() if len(p) else None)
    print("  first 20 idx", p[:20].tolist())
    print("  last 20 idx", p[-20:].tolist())
    print("  alpha of placed:", np.unique(tr.res["alpha"][p], return_counts=True))
