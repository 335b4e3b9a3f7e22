"""Generates the golden fixtures in tests/golden/ from the REFERENCE ITSELF
(oracle/_ref/libpythia_ref{16,64}.so = the unmodified reference sources compiled
by oracle/Makefile).  Run in the build container (needs /root/reference):

    make -C oracle && python tests/golden/make_golden.py
"""
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.py_oracle import Reference  # noqa: E402
from oracle.step import SEQ_COMMIT, SNAPSHOT, apply_warm_oracle, oracle_step, warm_ops  # noqa: E402
import test_oracle as T  # noqa: E402
from paper_2604_25899_b200 import workload as W  # noqa: E402


def enc(x):
    if isinstance(x, bytes):
        return {"b": x.hex()}
    if isinstance(x, (list, tuple)):
        return [enc(v) for v in x]
    if isinstance(x, (np.integer,)):
        return int(x)
    if isinstance(x, (np.floating, float)):
        return {"f": float(x).hex()}
    return x


def main():
    out = {"hashes": {}, "ops": {}, "routes": [], "steps": {}}
    rng = np.random.default_rng(2024)
    for B in (16, 64):
        ref = Reference(B)
        seqs = []
        for n in [0, 1, 15, 16, 17, 63, 64, 65, 150, 1000, 2049]:
            t = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2) + \
                rng.integers(0, 2, size=n, dtype=np.uint64)
            seqs.append({"tokens": t.tolist(), "hashes": ref.chain_hashes(t).tolist()})
        out["hashes"][str(B)] = seqs
        out["ops"][str(B)] = {str(seed): enc(T._random_ops(ref, seed, B, n_ops=120))
                              for seed in (101, 102)}
    ref = Reference(16)
    rr = np.random.default_rng(7)
    for _ in range(400):
        n = int(rr.integers(1, 40))
        spec = []
        for i in rr.permutation(n):
            k = int(rr.integers(0, 6))
            asg = [(int(rr.integers(0, 60)), int(rr.integers(0, 60)),
                    float(rr.choice([0.0, 1 - 0.99, 0.02])), int(rr.integers(0, 90)))
                   for _ in range(k)]
            spec.append((int(i), int(rr.integers(100, 500)), asg, int(rr.integers(0, 4))))
        req = (int(rr.integers(0, 60)), int(rr.integers(0, 60)), float(rr.choice([0.0, 1 - 0.99])),
               int(rr.integers(0, 60)))
        out["routes"].append({"spec": spec, "req": req, "decision": enc(T.route(ref, spec, req))})
    for B in (16, 64):
        ref = Reference(B)
        tr = W.deep_research(n_workflows=8, seed=31 + B, device="cpu")
        cl = W.make_cluster(6, 2, kv=20_000, l2=20_000, seed=B)
        caches = [ref.new_cache(int(cl.kv_capacity[n]), int(cl.l2_capacity[n]))
                  for n in range(cl.n_replicas)]
        l3, reg = ref.new_l3(), ref.new_registry()
        apply_warm_oracle(ref, caches, l3, reg, tr, warm_ops(tr, cl, 5))
        steps = []
        for s, mode in enumerate([SEQ_COMMIT, SEQ_COMMIT, SNAPSHOT]):
            o = oracle_step(ref, caches, l3, reg, tr, cl, mode, 0.05, 3.0 + s, True, True)
            dumps = [ref.dump(c, None, t).tobytes().hex() for c in caches for t in (0, 1)]
            dumps.append(ref.dump(caches[0], l3, 2).tobytes().hex())
            steps.append({"mode": mode, "decisions": enc(o["decisions"]),
                          "staged": o["staged"].tolist(), "placed": o["placed"],
                          "admitted": o["admitted"].tolist(), "match3": o["match3"].tolist(),
                          "dumps": dumps})
        out["steps"][str(B)] = {"workflows": 8, "seed": 31 + B, "cluster": [6, 2, 20_000, 20_000, B],
                                "warm_seed": 5, "steps": steps}
    with gzip.open(os.path.join(HERE, "reference_golden.json.gz"), "wt") as f:
        json.dump(out, f)
    print("wrote", os.path.join(HERE, "reference_golden.json.gz"))


if __name__ == "__main__":
    main()
