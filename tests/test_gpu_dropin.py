"""The drop-in (one call per reference call) path: pyg_lookup_all (the engine's node_view
loop in one launch) equals per-replica lookups, the memoized upload + hash of the last
sequence never serves stale tier state, and chain_hashes through the one-warp split task
equals the oracle for every block size."""
import numpy as np
import pytest

from oracle.py_oracle import Restated

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B", [16, 64, 5])
def test_lookup_all_equals_per_replica_lookups(B):
    from paper_2604_25899_b200 import Context
    rng = np.random.default_rng(B)
    n_rep = 6
    ctx = Context(n_rep, 1 << 40, 1 << 40, B)
    o = Restated(B)
    caches = [o.new_cache(1 << 40, 1 << 40) for _ in range(n_rep)]
    l3 = o.new_l3()
    base = rng.integers(1, 1 << 62, size=3000, dtype=np.uint64)
    prompts = [np.concatenate([base[:int(rng.integers(1, 3000))],
                               rng.integers(1, 1 << 62, size=int(rng.integers(0, 300)),
                                            dtype=np.uint64)]) for _ in range(12)]
    for k in range(40):
        p = prompts[int(rng.integers(0, len(prompts)))]
        n = int(rng.integers(0, n_rep))
        tier = int(rng.integers(0, 2))
        upto = int(rng.integers(0, len(p) + 1))
        ctx.insert_chain(n, tier, p, upto, 1, 1, float(k), 0)
        o.insert_chain(caches[n], tier, p, upto, 1, 1, float(k), 0)
        q = prompts[int(rng.integers(0, len(prompts)))]
        got = ctx.lookup_all(q, with_l3=True)
        for r in range(n_rep):
            assert tuple(got[r]) == tuple(ctx.lookup(r, q, with_l3=True)), (k, r)
            assert tuple(got[r]) == tuple(o.lookup(caches[r], l3, q)), (k, r)


def test_memoized_sequence_sees_fresh_tiers():
    from paper_2604_25899_b200 import Context
    B = 16
    rng = np.random.default_rng(3)
    ctx = Context(2, 1 << 40, 1 << 40, B)
    p = rng.integers(1, 1 << 62, size=777, dtype=np.uint64)
    assert ctx.lookup(0, p)[0] == 0
    ctx.insert_chain(0, 0, p, 400, 1, 1, 1.0, 0)          # same tokens: memo hit
    assert ctx.lookup(0, p)[0] == 400
    q = p.copy()
    q[500] ^= np.uint64(1)                                # same length, different content
    assert ctx.lookup(0, q)[0] == 400
    ctx.insert_chain(0, 0, q, len(q), 1, 1, 2.0, 0)
    assert ctx.lookup(0, q)[0] == len(q)
    assert ctx.lookup(0, p)[0] == 496                     # back to p: diverges at token 500
    o = Restated(B)
    for n in (1, 15, 16, 63, 64, 65, 511, 512, 513, 5000):
        s = rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
        assert np.array_equal(ctx.chain_hashes(s), o.chain_hashes(s)), n
