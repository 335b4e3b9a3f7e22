"""TEST INFRASTRUCTURE ONLY (parity checker + the reference CPU arm of bench.py).

The steady-state burst sequence of paper_2604_25899_b200/steady.py driven through the
UNMODIFIED reference (oracle/_ref/libpythia_ref{16,64}.so, oracle/ref_shim.cpp pref_burst /
pref_release):

  step k: release burst k-1's admitted requests of hold 1 and burst k-2's of hold 2
                                                          unpin_chain, hierarchy.cpp:132-142
          node table = background + burst k-1's placements of hold 2 (pool order,
                                                          engine.cpp:616-628)
          FutureRegistry updates of burst k's issue     engine.cpp:605-609
          pref_burst: node_view staged values, route with sequential commit, admission per
          replica in order against the live L3           engine.cpp:640-692, 799-829
"""
from __future__ import annotations

import numpy as np

from .py_oracle import RES_DTYPE, Reference
from .step import apply_warm_oracle

HOLD = 2


class RefSteady:
    def __init__(self, B, cl, threads=1, hash_once=True):
        self.ref = Reference(B)
        self.cl = cl
        self.caches = [self.ref.new_cache(int(cl.kv_capacity[n]), int(cl.l2_capacity[n]))
                       for n in range(cl.n_replicas)]
        self.l3, self.reg = self.ref.new_l3(), self.ref.new_registry()
        self.threads, self.hash_once = threads, hash_once
        self.hist = {}   # burst -> (tokens, tok_off, target replica index per request, admitted)

    def warm(self, trace, ops, fill_off, fill_placed, now=0.5):
        """The warm-up of steady.py: the warm fill, then the ops.  The fill runs while L2/L3
        are empty and every replica stays under its KV capacity, so admitting a placement
        (lookup, evict_for_space with nothing to free, insert_chain pinned) and releasing it
        is insert_chain(L1, prompt, len, lineage, now, 0) -- what this does, replica by
        replica in placement order (steady.apply_warm_fill_gpu runs the batched admission)."""
        n_fill = 0
        for n in range(self.cl.n_replicas):
            for r in fill_placed[fill_off[n]:fill_off[n + 1]]:
                p = trace.prompt(int(r))
                self.ref.insert_chain(self.caches[n], 0, p, len(p), int(trace.wf[r]),
                                      int(trace.role[r]), now, 0)
                n_fill += 1
        apply_warm_oracle(self.ref, self.caches, self.l3, self.reg, trace, ops)
        return n_fill

    def node_table(self, k):
        """background + burst k-1's placements still held (hold 2), per replica in placement
        order."""
        cl = self.cl
        base = [list(cl.asg[cl.asg_off[n]:cl.asg_off[n + 1]]) for n in range(cl.n_replicas)]
        if k - 1 in self.hist:
            _, _, tgt, _, res, hold = self.hist[k - 1]
            for r in np.nonzero((tgt >= 0) & (hold >= 2))[0]:
                base[int(tgt[r])].append(res[r])
        off = np.zeros(cl.n_replicas + 1, np.int64)
        np.cumsum([len(x) for x in base], out=off[1:])
        flat = [x for lst in base for x in lst]
        asg = np.array(flat, RES_DTYPE) if flat else np.zeros(0, RES_DTYPE)
        return off, asg

    def step(self, k, tokens, tok_off, res, group, wf, role, reg_wf, reg_mask, now, hold,
             want_staged=False):
        """hold: uint8 [R] bursts each request of this burst holds its replica (1 or 2)."""
        ref, cl = self.ref, self.cl
        for h in (1, 2):
            if k - h in self.hist:
                t, o, tgt, adm, _, hd = self.hist[k - h]
                ref.release(self.caches, t, o, tgt, (adm & (hd == h)).astype(np.int32))
        self.hist.pop(k - HOLD, None)
        off, asg = self.node_table(k)
        for w, m in zip(reg_wf.tolist(), reg_mask.tolist()):
            ref.reg_update(self.reg, int(w), int(m))
        dec, adm, m3, st = ref.burst(self.caches, self.l3, self.reg, True, tokens, tok_off, res,
                                     group, wf, role, cl.replica_id, cl.kv_capacity, off, asg,
                                     cl.cand_off, cl.cand, 0.05, now, self.hash_once,
                                     self.threads, want_staged)
        # replica_id == replica index in these clusters (make_cluster, id_base 0)
        tgt = dec["target"].astype(np.int32)
        self.hist[k] = (tokens, tok_off, tgt, adm.astype(np.int32), np.asarray(res, RES_DTYPE),
                        np.asarray(hold, np.uint8))
        return dec, adm, m3, st

    def dump(self, n, tier):
        return self.ref.dump(self.caches[n], self.l3 if tier == 2 else None, tier)
