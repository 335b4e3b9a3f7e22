"""K1 prefix memo on a synthetic batch: 40k requests of 4,096 tokens sharing 2,048-token
prefixes (64 distinct), memo on / off (profiles/r02_k1_prefix_memo_ab.txt)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2604_25899_b200 import Context
from paper_2604_25899_b200 import batch as PB
rng = np.random.default_rng(1)
R, L, P = 40000, 4096, 2048
pre = [rng.integers(0, 1 << 63, size=P, dtype=np.uint64) for _ in range(64)]
seqs = [np.concatenate([pre[i % 64], rng.integers(0, 1 << 63, size=L - P, dtype=np.uint64)]) for i in range(R)]
toks = np.concatenate(seqs)
off = np.arange(R + 1, dtype=np.int64) * L
for memo in (1, 0, 1, 0):
    ctx = Context(1, 1000, 1000, 16)
    ctx.set_hash_memo(memo)
    ctx.set_hash_split(0)
    z = np.zeros(R, np.int32)
    res = np.zeros(R, PB.RES_DTYPE)
    db = PB.upload_batch(ctx, toks, off, res, z, z, z)
    PB.bind_current_stream(ctx)
    ts = []
    for i in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); PB.hash_batch(ctx, db); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("synthetic memo", memo, "ms", sorted(ts)[2])
