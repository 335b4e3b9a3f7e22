"""Two pyg_ctx on two GPUs driven from ONE host thread whose current device is the other
one: every entry point must run on its ctx's device (PYG_ON_DEVICE), and K1's per-device
setup (shared-memory attribute, split-task constants) must hold on both."""
import numpy as np
import pytest
import torch

from oracle.py_oracle import Restated

pytestmark = pytest.mark.gpu


def test_two_ctxs_two_devices_one_thread():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    B = 16
    rng = np.random.default_rng(5)
    lens = np.concatenate([rng.integers(1, 3000, 200), [9000, 20000]])
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    toks = rng.integers(0, 1 << 62, size=int(off[-1]), dtype=np.uint64)
    z = np.zeros(len(lens), np.int32)
    res = np.zeros(len(lens), PB.RES_DTYPE)
    o = Restated(B)
    want = [o.chain_hashes(toks[off[r]:off[r + 1]]) for r in range(len(lens))]
    ctxs = [Context(2, 50_000, 50_000, B, device=d) for d in (0, 1)]
    for d in (1, 0):                     # current device = the OTHER one
        torch.cuda.set_device(1 - d)
        ctx = ctxs[d]
        dev = torch.device("cuda", d)
        db = PB.upload_batch(ctx, toks, off, res, z, z, z, device=dev)
        with torch.cuda.device(dev):
            PB.bind_current_stream(ctx)
        torch.cuda.set_device(1 - d)
        PB.hash_batch(ctx, db)
        torch.cuda.synchronize(dev)
        got = db.hashes.cpu().numpy().view(np.uint64)
        hoff = db.hash_off.cpu().numpy()
        for r in range(len(lens)):
            assert np.array_equal(got[hoff[r]:hoff[r + 1]], want[r]), (d, r)
        # drop-in calls (synchronous) on the ctx of the other device
        p = toks[off[3]:off[4]]
        ctx.insert_chain(1, 0, p, len(p), 7, 1, 1.0, 0)
        assert ctx.lookup(1, p)[0] == len(p)
        assert ctx.chain_hashes(p).tolist() == want[3].tolist()
    for c in ctxs:
        c.close()
