"""TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline composition).
Oracle composition of one batched step, and identical cluster-state builders
for the oracle and the GPU Context.  The step is the reference engine's call
pattern for a burst of requests (SURVEY.md CS-1 + CS-2):

  staged[r][j] = cache[cand_j].lookup(prompt_r, nullptr).l2     engine.cpp:646
  route(views, reservation_r, eps) for r in issue order          engine.cpp:650-692
      SEQ_COMMIT: the placement joins the target's pool before r+1
  per replica in order, per placed request in order: start_prefill cache side
      (lookup(seq,&l3) against the live L3, promoted spans erased at once,
       exactly the engine's one-at-a-time admission)              engine.cpp:799-829
  release: unpin_chain(seq, len) of admitted requests             hierarchy.cpp:132-142
"""
import numpy as np

from .py_oracle import RES_DTYPE

SNAPSHOT, SEQ_COMMIT = 0, 1


def oracle_step(o, caches, l3, reg, trace, cl, mode, eps, now, spec, release):
    R = trace.R
    prompts = [trace.prompt(r) for r in range(R)]
    maxc = int(np.max(np.diff(cl.cand_off)))
    staged = np.zeros((R, maxc), np.int32)
    for r in range(R):
        g = int(trace.group[r])
        cs = cl.cand[cl.cand_off[g]:cl.cand_off[g + 1]]
        for j, n in enumerate(cs):
            staged[r, j] = o.lookup(caches[n], None, prompts[r])[1]
    pools = [[tuple(cl.asg[k]) for k in range(cl.asg_off[n], cl.asg_off[n + 1])]
             for n in range(cl.n_replicas)]
    dec = []
    t_idx = np.full(R, -1, np.int32)
    for r in range(R):
        g = int(trace.group[r])
        cs = cl.cand[cl.cand_off[g]:cl.cand_off[g + 1]]
        rid = cl.replica_id[cs]
        cap = cl.kv_capacity[cs]
        off = [0]
        asg = []
        for n in cs:
            asg.extend(pools[n])
            off.append(len(asg))
        a = np.array(asg, RES_DTYPE) if asg else np.zeros(0, RES_DTYPE)
        req = tuple(trace.res[r])
        d = o.route(rid, cap, off, a, staged[r, :len(cs)].astype(np.int64), req, eps)
        dec.append(d)
        if d[0] >= 0:
            n = int(cs[list(rid).index(d[0])])
            t_idx[r] = n
            if mode == SEQ_COMMIT:
                pools[n].append(req)
    placed = [[r for r in range(R) if t_idx[r] == n] for n in range(cl.n_replicas)]
    admitted = np.zeros(R, np.int32)
    match3 = np.zeros((R, 3), np.int64)
    for n in range(cl.n_replicas):
        for r in placed[n]:
            # the live L3: a later admission no longer sees the L3 spans an earlier one
            # promoted (engine.cpp:806, 826-828; the engine admits one request at a time)
            ok, m = o.admit(caches[n], l3, l3, reg, spec, prompts[r], int(trace.wf[r]),
                            int(trace.role[r]), now)
            admitted[r] = int(ok)
            match3[r] = m
    if release:
        for n in range(cl.n_replicas):
            for r in placed[n]:
                if admitted[r]:
                    o.unpin_chain(caches[n], prompts[r], len(prompts[r]))
    return {"decisions": dec, "staged": staged, "placed": placed, "admitted": admitted,
            "match3": match3}


def warm_ops(trace, cl, seed=0, n_chains=6):
    """A deterministic list of warm-up ops: (kind, replica, args...)."""
    rng = np.random.default_rng(seed)
    ops = []
    for n in range(cl.n_replicas):
        for k in range(n_chains):
            r = int(rng.integers(0, trace.R))
            tier = int(rng.integers(0, 2))
            L = int(trace.tok_off[r + 1] - trace.tok_off[r])
            upto = L if rng.random() < 0.7 else int(rng.integers(0, L + 1))
            ops.append(("ins", n, tier, r, upto, int(trace.wf[r]), int(trace.role[r]),
                        float(rng.integers(0, 5)), 0))
    # write some lineages to L3 through the completion sweep
    for w in sorted(set(int(x) for x in rng.choice(trace.wf, 4))):
        ops.append(("cmp", w, int(rng.integers(0, 64)), 6.0))
    for w in sorted(set(int(x) for x in trace.wf)):
        ops.append(("reg", w, int(rng.integers(0, 64))))
    return ops


def apply_warm_oracle(o, caches, l3, reg, trace, ops):
    for op in ops:
        if op[0] == "ins":
            _, n, tier, r, upto, wf, role, now, pin = op
            o.insert_chain(caches[n], tier, trace.prompt(r), upto, wf, role, now, pin)
        elif op[0] == "cmp":
            _, w, mask, now = op
            for c in caches:
                o.complete(c, l3, w, mask, now)
            o.l3_dead_sweep(l3, w, mask)
        elif op[0] == "reg":
            o.reg_update(reg, op[1], op[2])
        elif op[0] == "l3put":  # TierStore::put into the shared L3 (hierarchy.cpp:44-66)
            _, r, upto, wf, role, now = op
            p = trace.prompt(r)
            B = o.B
            for i, h in enumerate(o.chain_hashes(p)):
                s0, e0 = i * B, min((i + 1) * B, len(p))
                if e0 > upto:
                    break
                o.put(caches[0], l3, 2, int(h), s0, e0, wf, role, now, 0)
        elif op[0] == "esp":
            _, n, tier, r, frm, to = op
            o.erase_chain_span(caches[n], None, tier, trace.prompt(r), frm, to)
        elif op[0] == "drop":
            o.reg_drop(reg, op[1])
        else:
            raise ValueError(op)


def apply_warm_gpu(ctx, trace, ops):
    for op in ops:
        if op[0] == "ins":
            _, n, tier, r, upto, wf, role, now, pin = op
            ctx.insert_chain(n, tier, trace.prompt(r), upto, wf, role, now, pin)
        elif op[0] == "cmp":
            _, w, mask, now = op
            for n in range(ctx.n_replicas):
                ctx.complete(n, w, mask, now)
            ctx.l3_dead_sweep(w, mask)
        elif op[0] == "reg":
            ctx.registry_update(op[1], op[2])
