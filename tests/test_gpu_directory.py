"""GPU parity of K2 through the L2 directory (csrc/k_dir.cu): the staged matrix of
every (request, candidate replica) pair must equal TierStore::matched_prefix on that
replica's L2 (hierarchy.cpp:84-104) as the oracle computes it.  Stress: many
replicas (1..4 mask words), shared prefixes with ragged tails, direct orphan puts
(short and > 63 tokens), erasures and re-puts between calls (stale directory),
zero-length prompts; walks on one thread, on one warp (forced with
PYG_K2_WARP_MIN=0) and mixed, with prompts up to ~100 blocks so a warp walk
spans several 32-boundary rounds."""
import numpy as np
import pytest
import torch

from oracle.py_oracle import Restated

pytestmark = pytest.mark.gpu


def _random_prompts(rng, n, base, B):
    out = []
    for _ in range(n):
        p = base[rng.integers(len(base))]
        cut = int(rng.integers(0, len(p) + 1))
        tail = rng.integers(1, 1 << 40, size=int(rng.integers(0, 3 * B)), dtype=np.uint64)
        out.append(np.concatenate([p[:cut], tail]).astype(np.uint64))
    out.append(np.zeros(0, np.uint64))
    return out


@pytest.mark.parametrize("warp_min", [None, "0", "2000000000"])
@pytest.mark.parametrize("n_rep,B,nb", [(5, 16, 12), (70, 16, 12), (200, 8, 12), (33, 64, 12),
                                        (40, 16, 100), (300, 8, 60)])
def test_staged_matrix_directory(n_rep, B, nb, warp_min, monkeypatch):
    if warp_min is not None:
        monkeypatch.setenv("PYG_K2_WARP_MIN", warp_min)
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    rng = np.random.default_rng(n_rep * 100 + B)
    o = Restated(B)
    caches = [o.new_cache(200_000, 200_000) for _ in range(n_rep)]
    ctx = Context(n_rep, [200_000] * n_rep, [200_000] * n_rep, B)
    base = [rng.integers(1, 1 << 40, size=int(rng.integers(1, nb * B)), dtype=np.uint64)
            for _ in range(12)]
    # L2 contents: prefixes of shared bases with ragged ends
    for n in range(n_rep):
        for _ in range(int(rng.integers(1, 6))):
            p = base[rng.integers(len(base))]
            upto = int(rng.integers(1, len(p) + 1))
            o.insert_chain(caches[n], 1, p, upto, 1, 1, 0.5, 0)
            ctx.insert_chain(n, 1, p, upto, 1, 1, 0.5, 0)
        if rng.random() < 0.3:  # orphan puts: short ragged and long
            p = base[rng.integers(len(base))]
            s = B * int(rng.integers(0, max(1, len(p) // B)))
            e = min(len(p), s + int(rng.integers(1, 80)))
            if e > s:
                h = int(o.chain_hashes(p[:e])[-1]) if e % B else int(rng.integers(1 << 62))
                o.put(caches[n], None, 1, h, s, e, 2, 2, 0.7, 0)
                ctx.put(n, 1, h, s, e, 2, 2, 0.7, 0)
    prompts = _random_prompts(rng, 300, base, B)
    off = np.zeros(len(prompts) + 1, np.int64)
    np.cumsum([len(p) for p in prompts], out=off[1:])
    toks = np.concatenate(prompts) if off[-1] else np.zeros(1, np.uint64)
    R = len(prompts)
    # candidate groups: all replicas, a strided subset (non-contiguous), a reversed subset
    groups = [list(range(n_rep)), list(range(0, n_rep, 3)), list(range(n_rep - 1, -1, -2))]
    cand_off = np.cumsum([0] + [len(g) for g in groups]).astype(np.int32)
    cand = np.concatenate(groups).astype(np.int32)
    grp = rng.integers(0, len(groups), R).astype(np.int32)
    res = np.zeros(R, PB.RES_DTYPE)
    db = PB.upload_batch(ctx, toks, off, res, grp, grp, grp)
    dn = PB.upload_nodes(np.arange(n_rep), np.full(n_rep, 10**6), np.zeros(n_rep + 1, np.int64),
                         np.zeros(0, PB.RES_DTYPE), cand_off, cand)
    out = PB.alloc_out(ctx, db, dn)

    def check():
        PB.bind_current_stream(ctx)
        PB.hash_batch(ctx, db)
        PB.staged_matrix(ctx, db, dn, out)
        torch.cuda.synchronize()
        ctx.check_device_error()
        got = out.staged.cpu().numpy()
        for r in range(R):
            g = groups[grp[r]]
            want = [o.matched_prefix(caches[n], None, 1, prompts[r]) for n in g]
            assert got[r, :len(g)].tolist() == want, (r, grp[r])
            assert not got[r, len(g):].any()

    check()
    # erase some blocks, re-put others: the directory must follow (stale -> rebuilt)
    for n in rng.choice(n_rep, min(n_rep, 6), replace=False):
        blocks = o.dump(caches[n], None, 1)
        for b in blocks[: max(1, len(blocks) // 3)]:
            o.erase(caches[n], None, 1, int(b["id"]))
            ctx.erase(int(n), 1, int(b["id"]))
    check()
