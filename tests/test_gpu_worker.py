"""GPU parity of K7 (csrc/k_worker.cu): form_batch and select_preemption_victim for many
replica queues at once, against the reference-pinned restatement (oracle/worker_oracle.py)."""
import numpy as np
import pytest
import torch

from oracle import worker_oracle as WO
from test_worker import random_queue

pytestmark = pytest.mark.gpu

QDT = np.dtype([("base", "<f8"), ("enq", "<f8"), ("res", "<i8"), ("id", "<i8")])


def test_form_batch_and_victim_many_queues():
    import ctypes as C
    from paper_2604_25899_b200 import Context, _lib
    rng = np.random.default_rng(5)
    sets = [random_queue(rng, int(n)) for n in rng.integers(1, 1500, 60)] + \
        [random_queue(rng, 4096), random_queue(rng, 1)]
    now, aging = 4.5, 0.02
    off = np.zeros(len(sets) + 1, np.int64)
    np.cumsum([len(s) for s in sets], out=off[1:])
    items = np.zeros(off[-1], QDT)
    for k, s in enumerate(sets):
        items[off[k]:off[k + 1]] = s
    act = rng.integers(0, 3000, len(sets)).astype(np.int64)
    cap = rng.integers(0, 400000, len(sets)).astype(np.int64)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).cuda()  # noqa: E731
    d_off, d_items, d_act, d_cap = d(off), d(items), d(act), d(cap)
    order = torch.zeros(int(off[-1]), dtype=torch.int32, device="cuda")
    nadm = torch.zeros(len(sets), dtype=torch.int32, device="cuda")
    vic = torch.zeros(len(sets), dtype=torch.int32, device="cuda")
    ctx = Context(1, 1000, 1000, 16)
    ctx.set_stream(None)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib._lib.pyg_form_batch_dev(ctx.h, len(sets), p(d_off), p(d_items), p(d_act),
                                            p(d_cap), now, aging, p(order), p(nadm)))
    _lib.check(_lib._lib.pyg_preemption_victim_dev(ctx.h, len(sets), p(d_off), p(d_items), now,
                                                   aging, p(vic)))
    torch.cuda.synchronize()
    ctx.check_device_error()
    o, na, v = order.cpu().numpy(), nadm.cpu().numpy(), vic.cpu().numpy()
    for k, s in enumerate(sets):
        want = WO.form_batch(s, int(act[k]), int(cap[k]), now, aging)
        assert na[k] == len(want), k
        assert list(o[off[k]:off[k] + na[k]]) == want, k
        assert v[k] == WO.preemption_victim(s, now, aging), k
