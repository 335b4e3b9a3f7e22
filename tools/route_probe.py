"""K3 cost probe (experiments): route a synthetic burst of R requests over G groups of 16
replicas (seq-commit), no cache state needed.  Prints the device time per call.
  python tools/route_probe.py R G [--staged]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_25899_b200 import Context  # noqa: E402
from paper_2604_25899_b200 import batch as PB  # noqa: E402
from paper_2604_25899_b200 import workload as W  # noqa: E402


def main():
    R, G = int(sys.argv[1]), int(sys.argv[2])
    rng = np.random.default_rng(0)
    cl = W.make_cluster(16 * G, G, seed=0)
    ctx = Context(16 * G, cl.kv_capacity, cl.l2_capacity, 16)
    res = np.zeros(R, PB.RES_DTYPE)
    res["prompt_len"] = rng.integers(500, 3000, R)
    res["upper"] = 1500
    res["alpha"] = np.where(rng.random(R) < 0.1, 0.0, 0.01)
    grp = rng.integers(0, G, R).astype(np.int32)
    dev = "cuda"
    t_res = torch.from_numpy(res.view(np.int64).reshape(R, 4).copy()).to(dev)
    t_grp = torch.from_numpy(grp).to(dev)
    dn = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, cl.cand_off, cl.cand)
    staged = torch.from_numpy(rng.integers(0, 64, (R, 16)).astype(np.int32)).to(dev)
    dec = torch.zeros((R, 3), dtype=torch.int64, device=dev)
    poff = torch.zeros(16 * G + 1, dtype=torch.int32, device=dev)
    pl = torch.zeros(R, dtype=torch.int32, device=dev)
    import ctypes as C
    from paper_2604_25899_b200 import _lib
    PB.bind_current_stream(ctx)
    ns = dn.struct()

    def call():
        _lib.check(_lib._lib.pyg_route_batch_dev(ctx.h, 1, C.byref(ns), C.c_void_p(t_res.data_ptr()),
                                                 R, C.c_void_p(t_grp.data_ptr()), G,
                                                 C.c_void_p(dn.cand_off.data_ptr()),
                                                 C.c_void_p(dn.cand.data_ptr()), dn.max_cand,
                                                 C.c_void_p(staged.data_ptr()), 0.05,
                                                 C.c_void_p(dec.data_ptr()),
                                                 C.c_void_p(poff.data_ptr()), C.c_void_p(pl.data_ptr())))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        call()
    b.record()
    torch.cuda.synchronize()
    print(f"R={R} G={G}: {a.elapsed_time(b) / 10:.3f} ms per route call, placed {int(poff[-1])}")


if __name__ == "__main__":
    main()
