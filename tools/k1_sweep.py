"""K1 alone on config-4 bursts of several sizes: split tasks on (default threshold) and off.
Prints one JSON line per (R, split_min): median ms of 7 launches (CUDA events on the ctx
stream), tokens, achieved GB/s of the K1 algorithmic bytes.

  python tools/k1_sweep.py [--sizes 1000,16000,125000]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1000,16000,125000")
    ap.add_argument("--splits", default="-1,8192,4096,0")
    ap.add_argument("--workload", default="bursty")
    ap.add_argument("--grids", default="persistent,tasks")
    ap.add_argument("--memo", default="1")
    a = ap.parse_args()
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import steady as S
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    for R in [int(x) for x in a.sizes.split(",")]:
        tr = S.make_burst(3, R, 1, dev, a.workload, 8)
        b = S.upload_burst(tr, 16, dev, 3)
        L = np.diff(tr.tok_off)
        nbytes = 8 * int(L.sum()) + 8 * b.b.n_hashes + 16 * (R + 1)
        for sm, grid, memo in [(int(x), gm, int(mm)) for x in a.splits.split(",")
                               for gm in a.grids.split(",") for mm in a.memo.split(",")]:
            ctx = Context(0, [], [], 16, device=0)
            ctx.set_hash_grid(grid)
            ctx.set_hash_memo(memo)
            ctx.set_stream(ctypes.c_void_p(s.cuda_stream))
            ctx.set_hash_split(sm)
            ts = []
            for i in range(9):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                PB.hash_batch(ctx, b.b)
                e1.record(s)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            print(json.dumps({"R": R, "split_min": sm, "grid": grid, "memo": memo, "ms": ms, "tokens": int(L.sum()),
                              "max_len": int(L.max()), "gbs": nbytes / ms / 1e6}), flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
