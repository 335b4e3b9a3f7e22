"""Multi-GPU step: replicas and their cache shards partitioned over the GPUs of one
box, one process per GPU.

Rank g owns global replicas [rep_off[g], rep_off[g+1]) -- their L1/L2 tiers live
only in rank g's pyg_ctx -- and receives requests [req_off[g], req_off[g+1]) of
the burst (global issue order = rank order, then index).  One step:

  1. K1  hash the local requests                        (local)
  2. K2  staged row of every local request against ALL its candidates, through the
         replicated L2 directory (one walk per request)  (local)
  3. NCCL all-gather of the per-request route inputs (reservation, group, length,
         lineage, staged row) -> every rank holds the whole burst's K3 inputs
  4. K3  sequential-commit route of the whole burst over the global node table,
         identically on every rank (engine.cpp:650-692 order; decisions bit-equal)
  5. NCCL all-to-all: each placed request's tokens and boundary hashes travel from
         its origin rank to the rank owning its target replica
  6. K4/K5 admission on the owner, per replica in global placement order
         (engine.cpp:799-829); it exports the L2 blocks it erases and the L3 chain
         hashes it promotes
  7. NCCL all-gather of those lists: every rank clears the directory bits and
         erases the union from its replica of the shared L3 (erasures commute)
  8. release (unpin) on the owner; admission results return to the origin (all-to-all)

Every collective carries data whose order is fixed by the global request order,
so the result is bit-identical to one GPU holding the whole cluster (and to the
oracle).  The index bookkeeping below is plain torch on whatever device the
tensors live on (tests run it on CPU with gloo); all hot-path compute is
libpyg_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import DEC_DTYPE, check

_PAYLOAD_FIXED = 14  # int32 words per request before the staged row


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class ShardPlan:
    """Static partition of replicas and requests over ranks."""

    def __init__(self, reps_per_rank, reqs_per_rank, rank, B):
        self.world = len(reps_per_rank)
        self.rank = rank
        self.B = B
        self.rep_off = np.concatenate([[0], np.cumsum(reps_per_rank)]).astype(np.int64)
        self.req_off = np.concatenate([[0], np.cumsum(reqs_per_rank)]).astype(np.int64)
        self.n_global = int(self.rep_off[-1])
        self.R_total = int(self.req_off[-1])
        self.rep_base = int(self.rep_off[rank])
        self.n_local = int(reps_per_rank[rank])
        self.req_base = int(self.req_off[rank])
        self.R_local = int(reqs_per_rank[rank])

    def owner(self, target: torch.Tensor) -> torch.Tensor:
        """rank owning each global replica id (-1 stays -1)."""
        bounds = torch.as_tensor(self.rep_off[1:-1], dtype=target.dtype, device=target.device)
        o = torch.bucketize(target, bounds, right=True)
        return torch.where(target >= 0, o, torch.full_like(o, -1))


def allgather_cat(t: torch.Tensor) -> torch.Tensor:
    """Concatenation of every rank's equal-shape tensor along dim 0 (rank order)."""
    ws = dist.get_world_size()
    if ws == 1:
        return t
    if dist.get_backend() == "nccl":
        out = torch.empty((ws * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous())
        return out
    parts = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(parts, t.contiguous())
    return torch.cat(parts)


def allgather_var(t: torch.Tensor, counts) -> torch.Tensor:
    """Variable-length all-gather: rank k contributes t[:counts[k]] (counts known everywhere);
    returns the concatenation in rank order."""
    ws = dist.get_world_size()
    if ws == 1:
        return t[:counts[0]]
    if len(set(counts)) == 1 and t.shape[0] == counts[0]:
        return allgather_cat(t)
    cap = max(max(counts), 1)
    buf = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    n = counts[dist.get_rank()]
    buf[:n] = t[:n]
    g = allgather_cat(buf)
    return torch.cat([g[k * cap:k * cap + counts[k]] for k in range(ws)])


def pack_payload(res_i64: torch.Tensor, group, wf, role, lens, staged) -> torch.Tensor:
    """Per-request route inputs as one int32 row: reservation (8 words), group, wf, role,
    pad, length (2 words), staged row."""
    R = res_i64.shape[0]
    fixed = torch.empty((R, _PAYLOAD_FIXED), dtype=torch.int32, device=res_i64.device)
    fixed[:, 0:8] = res_i64.contiguous().view(torch.int32).reshape(R, 8)
    fixed[:, 8] = group
    fixed[:, 9] = wf
    fixed[:, 10] = role
    fixed[:, 11] = 0
    fixed[:, 12:14] = lens.to(torch.int64).reshape(R, 1).view(torch.int32).reshape(R, 2)
    return torch.cat([fixed, staged.to(torch.int32)], dim=1)


def unpack_payload(p: torch.Tensor):
    R = p.shape[0]
    res = p[:, 0:8].contiguous().view(torch.int64).reshape(R, 4)
    lens = p[:, 12:14].contiguous().view(torch.int64).reshape(R)
    return (res, p[:, 8].contiguous(), p[:, 9].contiguous(), p[:, 10].contiguous(), lens,
            p[:, _PAYLOAD_FIXED:].contiguous())


@dataclass
class Dispatch:
    """Who sends which placed request where (all derived from the global decisions)."""
    send_idx: torch.Tensor      # int64 local request indices, destination-major, ascending
    send_counts: list           # requests per destination
    send_tok: list              # tokens per destination
    send_hash: list             # boundary hashes per destination
    recv_gidx: torch.Tensor     # int64 global indices of requests placed on my replicas, ascending
    recv_counts: list
    recv_tok: list
    recv_hash: list
    hash_to: list               # boundary hashes received by each rank (bounds its erase lists)


def dispatch_plan(plan: ShardPlan, target: torch.Tensor, lens: torch.Tensor) -> Dispatch:
    """target/lens over the whole burst (global order).  One device->host copy (G x G x 3)."""
    G, B = plan.world, plan.B
    dev = target.device
    owner = plan.owner(target.to(torch.int64))
    src = torch.bucketize(torch.arange(plan.R_total, device=dev),
                          torch.as_tensor(plan.req_off[1:-1], device=dev), right=True)
    ok = owner >= 0
    pair = (src * G + owner)[ok]
    nb = (lens + B - 1) // B
    cnt = torch.bincount(pair, minlength=G * G)
    tok = torch.bincount(pair, weights=lens[ok].to(torch.float64), minlength=G * G)
    hsh = torch.bincount(pair, weights=nb[ok].to(torch.float64), minlength=G * G)
    m = torch.stack([cnt.to(torch.float64), tok, hsh]).cpu().numpy().round().astype(np.int64)
    m = m.reshape(3, G, G)
    me = plan.rank
    lo, hi = plan.req_base, plan.req_base + plan.R_local
    own_l = owner[lo:hi]
    sel = torch.nonzero(own_l >= 0).flatten()
    order = torch.argsort(own_l[sel], stable=True)
    send_idx = sel[order]
    recv_gidx = torch.nonzero(owner == me).flatten()
    return Dispatch(send_idx, m[0, me].tolist(), m[1, me].tolist(), m[2, me].tolist(), recv_gidx,
                    m[0, :, me].tolist(), m[1, :, me].tolist(), m[2, :, me].tolist(),
                    m[2].sum(axis=0).tolist())


def local_placed(plan: ShardPlan, placed_off: torch.Tensor, placed: torch.Tensor,
                 recv_gidx: torch.Tensor):
    """Global per-replica placed lists (global request indices, placement order) -> the
    owner's per-local-replica lists of local batch indices."""
    a, b = plan.rep_base, plan.rep_base + plan.n_local
    off = placed_off[a:b + 1].to(torch.int64)
    vals = placed[int(off[0]):int(off[-1])].to(torch.int64) if off.numel() else placed[:0]
    loc = torch.searchsorted(recv_gidx, vals)
    return (off - off[0]).to(torch.int32), loc.to(torch.int32)


def a2a(send: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
    out = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype,
                      device=send.device)
    send = send[:sum(send_counts)]
    if dist.get_world_size() == 1:
        out.copy_(send)
        return out
    dist.all_to_all_single(out, send.contiguous(), recv_counts, send_counts)
    return out


def csr_offsets(lens: torch.Tensor) -> torch.Tensor:
    off = torch.zeros(lens.numel() + 1, dtype=torch.int64, device=lens.device)
    torch.cumsum(lens.to(torch.int64), 0, out=off[1:])
    return off


class ShardedStep:
    """One rank's side of the multi-GPU step (see module doc).  `nodes` is the global node
    table (every replica of the cluster, global candidate ids); `batch` holds this rank's
    requests."""

    def __init__(self, ctx, plan: ShardPlan, batch, nodes, device):
        from . import batch as PB
        self.PB = PB
        self.ctx, self.plan, self.b, self.nodes, self.dev = ctx, plan, batch, nodes, device
        check(_lib._lib.pyg_set_shard(ctx.h, plan.rep_base, plan.n_global))
        R, Rt, mc = plan.R_local, plan.R_total, max(nodes.max_cand, 1)
        self.staged = torch.zeros((max(R, 1), mc), dtype=torch.int32, device=device)
        self.decisions = torch.zeros((max(Rt, 1), 3), dtype=torch.int64, device=device)
        self.placed_off = torch.zeros(plan.n_global + 1, dtype=torch.int32, device=device)
        self.placed = torch.zeros(max(Rt, 1), dtype=torch.int32, device=device)
        self.counts = torch.zeros(2, dtype=torch.int64, device=device)
        self.lens = (batch.tok_off[1:] - batch.tok_off[:-1]).contiguous()
        self.req_counts = np.diff(plan.req_off).tolist()
        self.launches = 0

    # ---------------------------------------------------------------- directory
    def build_directory(self):
        """All-gather every shard's L2 records and (re)build the replicated directory."""
        cap = int(_lib._lib.pyg_dir_export_cap(self.ctx.h))
        rec = torch.empty((cap, 5), dtype=torch.int64, device=self.dev)  # 40-byte records
        n = C.c_int64()
        check(_lib._lib.pyg_dir_export_dev(self.ctx.h, _ptr(rec), cap, C.byref(n)))
        nt = torch.tensor([n.value], dtype=torch.int64, device=self.dev)
        counts = allgather_cat(nt).cpu().tolist()
        allrec = allgather_var(rec, counts)
        check(_lib._lib.pyg_dir_build_dev(self.ctx.h, _ptr(allrec), int(allrec.shape[0])))

    # ---------------------------------------------------------------- the step
    def step(self, now: float, speculative=True, release=True, mode=1, ev_hash=None,
             marks=None):
        """marks: optional list; (name, cuda event, host time) appended at phase ends."""
        ctx, plan, b, nodes, PB = self.ctx, self.plan, self.b, self.nodes, self.PB

        def mark(name):
            if marks is not None:
                import time
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append((name, e, time.perf_counter()))

        mark("start")
        PB.bind_current_stream(ctx)
        lib = _lib._lib
        # 1-2: local hash + staged rows
        if ev_hash:
            ev_hash[0].record()
        PB.hash_batch(ctx, b)
        if ev_hash:
            ev_hash[1].record()
        check(lib.pyg_staged_matrix_dev(ctx.h, _ptr(b.tokens), _ptr(b.tok_off), _ptr(b.hash_off),
                                        _ptr(b.hashes), plan.R_local, _ptr(b.group),
                                        nodes.n_groups, _ptr(nodes.cand_off), _ptr(nodes.cand),
                                        nodes.max_cand, _ptr(self.staged)))
        mark("hash+staged")
        # 3: all-gather route inputs
        pay = pack_payload(b.res[:plan.R_local], b.group[:plan.R_local], b.wf[:plan.R_local],
                           b.role[:plan.R_local], self.lens, self.staged[:plan.R_local])
        g_res, g_group, g_wf, g_role, g_lens, g_staged = unpack_payload(
            allgather_var(pay, self.req_counts))
        mark("allgather")
        # 4: route the whole burst (identical on every rank)
        ns = nodes.struct()
        check(lib.pyg_route_batch_dev(ctx.h, mode, C.byref(ns), _ptr(g_res), plan.R_total,
                                      _ptr(g_group), nodes.n_groups, _ptr(nodes.cand_off),
                                      _ptr(nodes.cand), nodes.max_cand, _ptr(g_staged), 0.05,
                                      _ptr(self.decisions), _ptr(self.placed_off),
                                      _ptr(self.placed)))
        target = self.decisions[:plan.R_total].view(torch.int32).reshape(-1, 6)[:, 0]
        mark("route")
        # 5: placed requests' tokens and hashes to their owners
        dp = dispatch_plan(plan, target, g_lens)
        s_lens = self.lens[dp.send_idx]
        s_nb = (s_lens + plan.B - 1) // plan.B
        s_toff, s_hoff = csr_offsets(s_lens), csr_offsets(s_nb)
        s_tok = torch.empty(max(int(sum(dp.send_tok)), 1), dtype=torch.int64, device=self.dev)
        s_hash = torch.empty(max(int(sum(dp.send_hash)), 1), dtype=torch.int64, device=self.dev)
        check(lib.pyg_gather_csr_dev(ctx.h, _ptr(b.tokens), _ptr(b.tok_off), _ptr(dp.send_idx),
                                     dp.send_idx.numel(), _ptr(s_toff), _ptr(s_tok)))
        check(lib.pyg_gather_csr_dev(ctx.h, _ptr(b.hashes), _ptr(b.hash_off), _ptr(dp.send_idx),
                                     dp.send_idx.numel(), _ptr(s_hoff), _ptr(s_hash)))
        r_tok = a2a(s_tok, dp.send_tok, dp.recv_tok)
        r_hash = a2a(s_hash, dp.send_hash, dp.recv_hash)
        mark("dispatch")
        # 6: admission of the requests placed on my replicas
        n_in = dp.recv_gidx.numel()
        l_lens = g_lens[dp.recv_gidx]
        l_toff = csr_offsets(l_lens)
        l_hoff = csr_offsets((l_lens + plan.B - 1) // plan.B)
        l_wf = g_wf[dp.recv_gidx].contiguous()
        l_role = g_role[dp.recv_gidx].contiguous()
        p_off, p_loc = local_placed(plan, self.placed_off, self.placed, dp.recv_gidx)
        adm = torch.zeros(max(n_in, 1), dtype=torch.int32, device=self.dev)
        m3 = torch.zeros((max(n_in, 1), 3), dtype=torch.int64, device=self.dev)
        cap = max(int(sum(dp.recv_hash)), 1)
        l2_out = torch.empty((cap, 5), dtype=torch.int64, device=self.dev)
        l3_out = torch.empty(cap, dtype=torch.int64, device=self.dev)
        p_loc = p_loc if p_loc.numel() else torch.zeros(1, dtype=torch.int32, device=self.dev)
        check(lib.pyg_admit_shard_dev(ctx.h, _ptr(r_tok), _ptr(l_toff), _ptr(l_hoff),
                                      _ptr(r_hash), _ptr(l_wf), _ptr(l_role), n_in, _ptr(p_off),
                                      _ptr(p_loc), now, int(bool(speculative)), _ptr(adm),
                                      _ptr(m3), _ptr(l2_out), cap, _ptr(l3_out), cap,
                                      _ptr(self.counts)))
        mark("admit")
        # 7: every shard applies every shard's L2-directory clears and L3 erasures
        caps = [max(int(x), 1) for x in dp.hash_to]
        g_cnt = allgather_cat(self.counts.reshape(1, 2))
        cmax = max(caps)
        buf = torch.zeros((cmax, 6), dtype=torch.int64, device=self.dev)
        buf[:cap, :5] = l2_out
        buf[:cap, 5] = l3_out
        g_buf = allgather_cat(buf)
        for k in range(plan.world):
            blk = g_buf[k * cmax:(k + 1) * cmax]
            l2k = blk[:, :5].contiguous()
            l3k = blk[:, 5].contiguous()
            if k != plan.rank:
                check(lib.pyg_dir_clear_dev(ctx.h, _ptr(l2k), cmax, _ptr(g_cnt[k, 0:1])))
            check(lib.pyg_l3_erase_hashes_dev(ctx.h, _ptr(l3k), cmax, _ptr(g_cnt[k, 1:2])))
        mark("l2l3_lists")
        # 8: release, results back to the origins
        if release and n_in:
            check(lib.pyg_release_batch_dev(ctx.h, _ptr(l_toff), _ptr(l_hoff), _ptr(r_hash), n_in,
                                            _ptr(p_off), _ptr(p_loc), _ptr(adm)))
        back = torch.cat([adm[:n_in].to(torch.int64).reshape(-1, 1), m3[:n_in]], dim=1)
        ret = a2a(back.contiguous(), dp.recv_counts, dp.send_counts)
        out_adm = torch.zeros(max(plan.R_local, 1), dtype=torch.int32, device=self.dev)
        out_m3 = torch.zeros((max(plan.R_local, 1), 3), dtype=torch.int64, device=self.dev)
        if ret.shape[0]:
            out_adm[dp.send_idx] = ret[:, 0].to(torch.int32)
            out_m3[dp.send_idx] = ret[:, 1:]
        mark("release+return")
        return {"decisions": self.decisions[:plan.R_total], "placed_off": self.placed_off,
                "placed": self.placed, "admitted": out_adm[:plan.R_local],
                "match3": out_m3[:plan.R_local], "staged": self.staged[:plan.R_local],
                "n_placed_here": n_in}


def decisions_host(dec: torch.Tensor) -> np.ndarray:
    return dec.cpu().numpy().view(DEC_DTYPE).reshape(-1)
