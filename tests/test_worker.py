"""Worker batch formation / preemption oracle (oracle/worker_oracle.py) pinned against the
compiled reference (sched/worker.cpp through oracle/ref_shim.cpp) on random queues with
heavy priority / enqueue-time ties."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import worker_oracle as WO

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libpythia_ref64.so")


def random_queue(rng, n):
    base = rng.choice([0.0, 0.5, 1.0, 1.25, -0.0], n) * rng.choice([1.0, 0.3], n)
    enq = rng.choice([0.0, 1.0, 1.5, 2.25, 3.0], n)
    res = rng.integers(0, 5000, n)
    ids = rng.permutation(10 * n)[:n]
    return [(float(base[i]), float(enq[i]), int(res[i]), int(ids[i])) for i in range(n)]


def _ref():
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(REF)
    lib.pref_form_batch.restype = C.c_int64
    lib.pref_preemption_victim.restype = C.c_int32
    return lib


def test_restatement_matches_reference():
    lib = _ref()
    rng = np.random.default_rng(11)
    for t in range(400):
        n = int(rng.integers(1, 60))
        q = random_queue(rng, n)
        now, aging = float(rng.choice([3.0, 5.5])), float(rng.choice([0.0, 0.02, 1.0]))
        base = np.array([x[0] for x in q]); enq = np.array([x[1] for x in q])
        res = np.array([x[2] for x in q], np.int64); ids = np.array([x[3] for x in q], np.int64)
        act, cap = int(rng.integers(0, 4000)), int(rng.integers(0, 40000))
        out = np.zeros(n, np.int32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        k = lib.pref_form_batch(n, p(base), p(enq), p(res), p(ids), C.c_int64(act), C.c_int64(cap),
                                C.c_double(now), C.c_double(aging), p(out))
        assert list(out[:k]) == WO.form_batch(q, act, cap, now, aging), t
        v = lib.pref_preemption_victim(n, p(base), p(enq), p(res), p(ids), C.c_double(now),
                                       C.c_double(aging))
        assert v == WO.preemption_victim(q, now, aging), t
