"""Steady-state burst stepping: the hot path run the way a serving loop runs it.

A trace arrives as successive bursts (windows of the issue order).  Step k handles burst k
on a cluster whose state carries over from the bursts before it:

  1. completions: a placed request holds its replica for hold(r) in {1, 2} bursts (by the
     parity of its global request id); at step k the admitted requests of burst k-1 with
     hold 1 and of burst k-2 with hold 2 are released         (unpin_chain,
     hierarchy.cpp:132-142; their blocks stay in L1, unpinned, so L1 fills and later
     admissions evict)
  2. node table of burst k: background load + the reservations of burst k-1's placements
     still held (hold 2), in pool order                       (engine.cpp:616-628, 686)
  3. FutureRegistry updates of burst k's issue (engine.cpp:605-609)
  4. K2 staged matrix -> K3 sequential-commit route -> K4/K5 admission with eviction and
     the ordered L3 promotion (engine.cpp:640-692, 799-829)
K1 (chain hashing) of burst k+1 runs on its own stream meanwhile (bench.py).

oracle/steady_ref.py drives the unmodified reference through the identical sequence;
bench.py --check compares the two burst by burst.  Everything here is plumbing (torch
buffers, index arrays); the compute is libpyg_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import batch as PB
from . import workload as W
from ._lib import check

HOLD = 2           # longest hold: a placement of burst k completes at step k+1 or k+2
N_MODELS = 8       # config 4 cluster: 8 models x 32 replicas = 256 replicas
REPLICAS = 256


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def registry_mask(role: np.ndarray) -> np.ndarray:
    """Issue-time future-role set of a bursty request (synthetic workflow shape): its own role
    and two later ones, so a workflow's blocks of other roles are dead (evicted first)."""
    r = role.astype(np.uint64)
    one = np.uint64(1)
    return (one << r) | (one << ((r + np.uint64(3)) % np.uint64(16))) | \
        (one << ((r + np.uint64(7)) % np.uint64(16)))


def hold_of(k: int, R: int, n: int) -> np.ndarray:
    """Bursts each request of burst k (R requests per burst; the first n) holds its
    replica once placed: 1 + parity of its global request id."""
    return (1 + ((k * R + np.arange(n)) & 1)).astype(np.uint8)


def registry_pairs(wf: np.ndarray, role: np.ndarray):
    """(distinct workflows, mask of their LAST request in issue order) -- the registry state
    after a burst's issue-time updates (update replaces the set)."""
    rev = wf[::-1]
    u, first_rev = np.unique(rev, return_index=True)
    last = len(wf) - 1 - first_rev
    return u.astype(np.int32), registry_mask(role[last])


def make_burst(k, R, seed=1, device="cuda", kind="bursty", n_models=N_MODELS, n_keep=None,
               **kw) -> W.Trace:
    """Burst k of a trace, R requests (request and workflow ids continue across bursts;
    prefixes / carried contexts are shared by the whole trace).  kind: 'bursty' (config 4)
    or 'long_context' (config 3).  n_keep: only the first n_keep requests of the burst."""
    if kind == "bursty":
        return W.bursty(n_requests=R, seed=seed * 1_000_003 + k, device=device,
                        n_models=n_models, r_base=k * R, n_keep=n_keep, **kw)
    if kind == "long_context":
        return W.long_context(n_requests=R, seed=seed * 1_000_003 + k, device=device,
                              r_base=k * R, n_keep=n_keep, **kw)
    raise ValueError(kind)


def make_bursts(n_bursts, R, seed=1, device="cuda", n_models=N_MODELS, first=0, kind="bursty",
                n_keep=None, **kw):
    """Bursts first .. first+n_bursts-1 (make_burst)."""
    return [make_burst(k, R, seed, device, kind, n_models, n_keep, **kw)
            for k in range(first, first + n_bursts)]


def config4_cluster(kv=100_000, l2=200_000, seed=0, n_replicas=REPLICAS, n_models=N_MODELS):
    """Config 4 cluster: models own contiguous replica blocks (8 x 32 by default), 0-3
    background reservations per replica."""
    return W.make_cluster(n_replicas, n_models, kv=kv, l2=l2, seed=seed)


@dataclass
class Burst:
    """One burst resident in HBM (+ the host arrays the bookkeeping needs)."""
    b: PB.DeviceBatch
    tok_off: np.ndarray
    res: np.ndarray
    group: np.ndarray
    wf: np.ndarray
    role: np.ndarray
    reg_wf: torch.Tensor
    reg_mask: torch.Tensor
    n_reg: int
    max_wf: int
    hold: torch.Tensor        # uint8 [R], bursts a placement is held (hold_of)
    hold_h: np.ndarray

    @property
    def R(self):
        return self.b.R


def upload_burst(tr: W.Trace, B: int, device, k: int = 0, R_full: int = 0) -> Burst:
    """Burst k of R_full requests per burst (tr may be its first tr.R requests)."""
    tok = tr.tokens if tr.tokens.device == torch.device(device) else tr.tokens.to(device)
    nb = (np.diff(tr.tok_off) + B - 1) // B
    hoff = np.zeros(tr.R + 1, np.int64)
    np.cumsum(nb, out=hoff[1:])
    db = PB.DeviceBatch(tr.R, tok, torch.from_numpy(tr.tok_off).to(device),
                        torch.from_numpy(hoff).to(device),
                        torch.empty(max(int(hoff[-1]), 1), dtype=torch.int64, device=device),
                        torch.from_numpy(tr.res.view(np.int64).reshape(tr.R, 4).copy()).to(device),
                        torch.from_numpy(tr.group).to(device), torch.from_numpy(tr.wf).to(device),
                        torch.from_numpy(tr.role).to(device), int(hoff[-1]), tr.n_tokens)
    rw, rm = registry_pairs(tr.wf, tr.role)
    hold = hold_of(k, R_full or tr.R, tr.R)
    return Burst(db, tr.tok_off, tr.res, tr.group, tr.wf, tr.role,
                 torch.from_numpy(rw).to(device), torch.from_numpy(rm.view(np.int64)).to(device),
                 len(rw), int(tr.wf.max()) if tr.R else 0, torch.from_numpy(hold).to(device),
                 hold)


class Steady:
    """The device side of the steady-state step on one GPU (ctx holds every replica)."""

    def __init__(self, ctx: _lib.Context, cl: W.Cluster, R_max: int, device):
        self.ctx, self.cl, self.dev = ctx, cl, device
        self.nodes = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg,
                                     cl.cand_off, cl.cand, device=device)
        # the node table the route reads: base + one burst's placements (<= R_max)
        self.base_off, self.base = self.nodes.asg_off, self.nodes.asg
        A = int(cl.asg_off[-1])
        self.nodes.asg_off = torch.zeros_like(self.base_off)
        self.nodes.asg = torch.zeros((A + R_max + 1, 4), dtype=torch.int64, device=device)
        dummy = PB.DeviceBatch(R_max, None, None, None, None, None, None, None, None, 0, 0)
        self.reserved_wf = -1
        self.outs = [PB.alloc_out(ctx, dummy, self.nodes, device=device) for _ in range(HOLD + 1)]
        self.placed_total = 0

    def out(self, k) -> PB.StepOut:
        return self.outs[k % (HOLD + 1)]

    def complete(self, bursts, k):
        """Step k's completions: burst k-1's admitted requests of hold 1, burst k-2's of
        hold 2 (bursts indexable by burst number)."""
        for h in (1, 2):
            if k - h < 0:
                continue
            b, o = bursts[k - h], self.out(k - h)
            check(_lib._lib.pyg_release_hold_dev(self.ctx.h, _ptr(b.b.tok_off),
                                                 _ptr(b.b.hash_off), _ptr(b.b.hashes), b.R,
                                                 _ptr(o.placed_off), _ptr(o.placed),
                                                 _ptr(o.admitted), _ptr(b.hold), h, None))

    def compose_nodes(self, prev: Burst | None, k):
        """node table of step k: base + burst k-1's placements still held (hold 2)."""
        o = self.out(k - 1) if prev is not None else None
        check(_lib._lib.pyg_nodes_compose_dev(
            self.ctx.h, self.cl.n_replicas, _ptr(self.base_off), _ptr(self.base),
            _ptr(o.placed_off) if o else None, _ptr(o.placed) if o else None,
            _ptr(prev.b.res) if prev else None, _ptr(prev.hold) if prev else None, 2,
            _ptr(self.nodes.asg_off), _ptr(self.nodes.asg)))

    def reserve(self, bursts):
        """Size the device registry for every burst's workflows up front (a growth inside the
        step would synchronize)."""
        mx = max(b.max_wf for b in bursts)
        if mx > self.reserved_wf:
            self.ctx.registry_reserve(mx)
            self.reserved_wf = mx

    def registry(self, burst: Burst):
        check(_lib._lib.pyg_registry_update_batch_dev(self.ctx.h, burst.n_reg, _ptr(burst.reg_wf),
                                                      _ptr(burst.reg_mask), burst.max_wf))

    def route_admit(self, burst: Burst, k, now, events=None, after_staged=None):
        """K2 -> K3 -> K4/K5 of burst k (its hashes are ready).  events: optional list of 4
        CUDA events recorded before K2, K3, admission and after it; after_staged() is called
        once K2 is enqueued (the bench starts the next burst's K1 there)."""
        o = self.out(k)
        rec = (lambda i: events[i].record()) if events else (lambda i: None)
        rec(0)
        PB.staged_matrix(self.ctx, burst.b, self.nodes, o)
        if after_staged is not None:
            after_staged()
        rec(1)
        PB.route_batch(self.ctx, burst.b, self.nodes, o, PB.SEQ_COMMIT)
        rec(2)
        PB.admit_batch(self.ctx, burst.b, o, now, True)
        rec(3)
        return o

    def step(self, k, bursts, now, events=None):
        """Everything of step k after K1 (bursts[k].b.hashes ready); bursts is indexable by
        burst number for k-2 .. k."""
        PB.bind_current_stream(self.ctx)
        self.complete(bursts, k)
        self.compose_nodes(bursts[k - 1] if k >= 1 else None, k)
        self.registry(bursts[k])
        return self.route_admit(bursts[k], k, now, events)


def warm_ops(warm: W.Trace, cl: W.Cluster, l3_prefixes=128, l2_per_group=64, seed=0):
    """Deterministic warm-up ops (oracle.step op format):
      ("ins", replica, 1, r, upto, wf, role, now, 0): request r's blocks up to `upto` staged
          into a replica's L2 (forward staging, manager.cpp:60-100) -- the first half of a
          few requests per group, spread over the group's replicas;
      ("l3put", r, upto, wf, role, now): the same chain blocks put straight into the shared
          L3 store (TierStore::put, hierarchy.cpp:44-66), as the completion sweep's
          RetainAndWriteL3 does (manager.cpp:44-58) -- identical on every GPU's replica."""
    rng = np.random.default_rng(seed)
    L = np.diff(warm.tok_off)
    ops = []
    for g in range(len(cl.cand_off) - 1):
        cands = cl.cand[cl.cand_off[g]:cl.cand_off[g + 1]]
        rs = np.nonzero(warm.group == g)[0][:l2_per_group]
        for i, r in enumerate(rs):
            rep = int(cands[i % len(cands)])
            upto = int(min(L[r], max(64, L[r] // 2)))
            ops.append(("ins", rep, 1, int(r), upto, int(warm.wf[r]), int(warm.role[r]), 0.25, 0))
    carrier = 1 << 28
    for r in rng.choice(warm.R, size=min(l3_prefixes, warm.R), replace=False):
        upto = int(min(L[r], max(64, L[r] // 2)))
        ops.append(("l3put", int(r), upto, carrier, 1, 0.75))
    return ops


def chain_blocks(hashes: np.ndarray, n: int, upto: int, B: int):
    """(hash, span_start, span_end) of the blocks insert_chain(tokens, upto) puts
    (hierarchy.cpp:119-130): boundary i spans [iB, min((i+1)B, n)) and stops past upto."""
    out = []
    for i, h in enumerate(hashes):
        s, e = i * B, min((i + 1) * B, n)
        if e > upto:
            break
        out.append((int(h), s, e))
    return out


def apply_ops_gpu(ctx, trace: W.Trace, ops, rep_base=0):
    """Apply warm_ops through the drop-in API (one call per op).  Sharded: this ctx holds
    global replicas [rep_base, rep_base + ctx.n_replicas); ops on other replicas are
    skipped, L3 ops (the replicated shared L3) always apply."""
    for op in ops:
        k = op[0]
        if k == "ins":
            _, n, tier, r, upto, wf, role, now, pin = op
            if rep_base <= n < rep_base + ctx.n_replicas:
                ctx.insert_chain(n - rep_base, tier, trace.prompt(r), upto, wf, role, now, pin)
        elif k == "l3put":
            _, r, upto, wf, role, now = op
            p = trace.prompt(r)
            for h, s0, e0 in chain_blocks(ctx.chain_hashes(p), len(p), upto, ctx.B):
                ctx.put(0, 2, h, s0, e0, wf, role, now, 0)
        elif k == "reg":
            ctx.registry_update(op[1], op[2])
        else:
            raise ValueError(op)


def warm_fill_plan(warm: W.Trace, cl: W.Cluster, fill_frac=0.9):
    """Placed CSR of the warm fill: warm requests assigned round-robin to their group's
    replicas until each replica's assigned tokens reach fill_frac of its KV capacity.  Admitted
    (pinned) then released, this leaves every L1 near full of unpinned blocks."""
    L = np.diff(warm.tok_off)
    load = np.zeros(cl.n_replicas, np.int64)
    lists = [[] for _ in range(cl.n_replicas)]
    nxt = {}
    for r in range(warm.R):
        g = int(warm.group[r])
        cands = cl.cand[cl.cand_off[g]:cl.cand_off[g + 1]]
        if len(cands) == 0:
            continue
        for _ in range(len(cands)):
            i = nxt.get(g, 0)
            nxt[g] = (i + 1) % len(cands)
            n = int(cands[i])
            if load[n] + L[r] <= fill_frac * cl.kv_capacity[n]:
                lists[n].append(r)
                load[n] += L[r]
                break
    off = np.zeros(cl.n_replicas + 1, np.int32)
    np.cumsum([len(x) for x in lists], out=off[1:])
    placed = np.concatenate([np.asarray(x, np.int32) for x in lists]) if off[-1] else \
        np.zeros(0, np.int32)
    return off, placed


def apply_warm_fill_gpu(ctx, warm: W.Trace, off, placed, B, device, now=0.5):
    """Admit the warm placements (K4/K5: lookup, evict, insert pinned) and release them.  Run
    it first, on empty tiers (then warm_ops): every replica stays under its KV capacity, so
    this leaves exactly insert_chain(L1, prompt, len, lineage, now, 0) per placement."""
    wb = upload_burst(warm, B, device, 0)
    PB.bind_current_stream(ctx)
    PB.hash_batch(ctx, wb.b)
    o = PB.StepOut(torch.zeros((warm.R, 3), dtype=torch.int64, device=device),
                   torch.zeros((1, 1), dtype=torch.int32, device=device),
                   torch.from_numpy(off).to(device),
                   torch.from_numpy(np.concatenate([placed, np.zeros(max(0, warm.R - len(placed)),
                                                                     np.int32)])).to(device),
                   torch.zeros(warm.R, dtype=torch.int32, device=device),
                   torch.zeros((warm.R, 3), dtype=torch.int64, device=device))
    PB.admit_batch(ctx, wb.b, o, now, True)
    PB.release_batch(ctx, wb.b, o)
    torch.cuda.synchronize(device)
    ctx.check_device_error()
    return int(o.admitted.sum().item())
