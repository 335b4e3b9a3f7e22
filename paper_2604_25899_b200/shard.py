"""Multi-GPU step: replicas and their cache shards partitioned over the GPUs of one
box, one process per GPU.

Rank g owns global replicas [rep_off[g], rep_off[g+1]) -- their L1/L2 tiers live
only in rank g's pyg_ctx -- and receives requests [req_off[g], req_off[g+1]) of
the burst (global issue order = rank order, then index).  One step:

  1. K1  hash the local requests                        (local)
  2. K2  staged row of every local request against ALL its candidates, through the
         replicated L2 directory (one walk per request)  (local)
  3. exchange of compact per-request route rows (tokens(), alpha, group, 16-bit staged
         row: 52 B at 16 candidates): each rank packs its rows into a double-buffered
         window, signals every peer through a flag array in peer memory, waits for all
         of them and reads their rows in place over NVLink -> every rank holds the whole
         burst's K3 inputs (PYG_SHARD_NCCL=1: NCCL all-gather instead)
  4. K3  sequential-commit route of the whole burst over the global node table,
         identically on every rank (engine.cpp:650-692 order; decisions bit-equal)
  5. the owner of each target replica PULLS the placed requests' tokens and boundary
         hashes out of the origin GPU's HBM over NVLink (CUDA IPC peer mappings set up
         once; csrc/k_shard.cu) -- sizes bounded by capacity_holds, counts on device
  6. K4/K5 admission on the owner, per replica in global placement order
         (engine.cpp:799-829); it exports the L2 blocks it erases
  7. the L3 promotions in engine order, chained over the ranks: rank g waits for
         the L3 erase lists of ranks < g (their admissions come first), applies them
         to its replica of the shared L3, resolves its own admissions' L3 matches in
         order and publishes its list; then every rank applies the remaining lists
         and clears the directory bits of every other rank's L2 erasures
  8. release (unpin) on the owner; each origin reads its requests' admission results
         from the owners (peer loads).  No host synchronisation inside the step.

Every collective carries data whose order is fixed by the global request order,
so the result is bit-identical to one GPU holding the whole cluster (and to the
oracle).  The index bookkeeping below is plain torch on whatever device the
tensors live on (tests run it on CPU with gloo); all hot-path compute is
libpyg_b200.so.
"""
from __future__ import annotations

import ctypes as C
import os
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


def csr_offsets(lens: torch.Tensor) -> torch.Tensor:
    off = torch.zeros(lens.numel() + 1, dtype=torch.int64, device=lens.device)
    torch.cumsum(lens.to(torch.int64), 0, out=off[1:])
    return off


WINDOW_FIELDS = ("tokens", "tok_off", "hashes", "hash_off", "recv_gidx", "recv_count", "admitted",
                 "match3", "l2_list", "l3_list", "list_counts", "workflow", "role")  # == pyg_peer


def exchange_windows(local_ptrs, export, import_):
    """Every rank publishes its exchange window (IPC handle + offset per field, pyg_peer
    order); returns, per rank, the field pointers valid in THIS process (own window: local
    pointers; others: imported peer mappings)."""
    mine = [export(p) for p in local_ptrs]
    ws = dist.get_world_size() if dist.is_initialized() else 1
    allw = [None] * ws
    if ws > 1:
        dist.all_gather_object(allw, mine)
    else:
        allw = [mine]
    me = dist.get_rank() if ws > 1 else 0
    return [list(local_ptrs) if k == me else [import_(h, o) for h, o in allw[k]]
            for k in range(ws)]


def barrier_on_stream(dev):
    """Cross-GPU stream barrier: a one-element NCCL all-reduce completes on this stream only
    after every rank's stream has reached it."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(torch.zeros(1, dtype=torch.int32, device=dev))


class ShardedStep:
    """One rank's side of the multi-GPU step (see module doc).  `nodes` is the global node
    table (every replica of the cluster, global candidate ids); `batch` holds this rank's
    requests.  Buffers other ranks read (inputs, receive lists, results, erase lists) are
    mapped into every peer with CUDA IPC once, here."""

    def __init__(self, ctx, plan: ShardPlan, batch, nodes, device, kv_capacity_local,
                 tokens_total=None):
        from . import batch as PB
        self.PB = PB
        self.ctx, self.plan, self.b, self.nodes, self.dev = ctx, plan, batch, nodes, device
        check(_lib._lib.pyg_set_shard(ctx.h, plan.rep_base, plan.n_global))
        R, Rt, mc, B = plan.R_local, plan.R_total, max(nodes.max_cand, 1), plan.B
        i32, i64 = torch.int32, torch.int64
        z = lambda *sh, dt=i64: torch.zeros(sh, dtype=dt, device=device)  # noqa: E731
        self.staged = z(max(R, 1), mc, dt=i32)
        self.decisions = z(max(Rt, 1), 3)
        self.placed_off = z(plan.n_global + 1, dt=i32)
        self.placed = z(max(Rt, 1), dt=i32)
        self.lens = (batch.tok_off[1:] - batch.tok_off[:-1]).contiguous()
        self.req_counts = np.diff(plan.req_off).tolist()
        # receive-side bounds: placed prompt tokens on a replica <= its kv_capacity
        kv = int(np.sum(kv_capacity_local))
        tt = int(tokens_total) if tokens_total is not None else kv + 1
        self.cap_req = max(1, min(Rt, kv))
        self.cap_tok = max(1, min(tt, kv + 1))
        self.cap_hash = self.cap_tok // B + self.cap_req + 1
        self.recv_gidx = z(self.cap_req, dt=i32)
        self.recv_count = z(1)
        self.recv_wf = z(self.cap_req, dt=i32)
        self.recv_role = z(self.cap_req, dt=i32)
        self.recv_toff = z(self.cap_req + 1)
        self.recv_hoff = z(self.cap_req + 1)
        self.r_tok = z(self.cap_tok)
        self.r_hash = z(self.cap_hash)
        self.adm = z(self.cap_req, dt=i32)
        self.m3 = z(self.cap_req, 3)
        self.l2_list = z(self.cap_hash, 5)
        self.l3_list = z(self.cap_hash)
        self.counts = z(2)
        self.p_off = z(plan.n_local + 1, dt=i32)
        self.p_loc = z(self.cap_req, dt=i32)
        self.out_adm = z(max(R, 1), dt=i32)
        self.out_m3 = z(max(R, 1), 3)
        self.rep_off_d = torch.as_tensor(plan.rep_off, dtype=i64, device=device)
        self.req_off_d = torch.as_tensor(plan.req_off, dtype=i64, device=device)
        local = [batch.tokens, batch.tok_off, batch.hashes, batch.hash_off, self.recv_gidx,
                 self.recv_count, self.adm, self.m3, self.l2_list, self.l3_list, self.counts,
                 batch.wf, batch.role]
        lib = _lib._lib

        def export(t):
            h = (C.c_char * 64)()
            off = C.c_int64()
            check(lib.pyg_ipc_export(C.c_void_p(t), h, C.byref(off)))
            return bytes(h), off.value

        def import_(h, off):
            p = C.c_void_p()
            check(lib.pyg_ipc_import(ctx.h, h, off, C.byref(p)))
            return p.value

        wins = exchange_windows([t.data_ptr() for t in local], export, import_)
        self.peers = torch.tensor(wins, dtype=torch.int64, device=device)  # [world, 13]
        # compact route rows: 16-bit staged values when every prompt of the burst is < 64k
        lmax = torch.zeros(1, dtype=torch.int64, device=device)
        if R:
            lmax[0] = self.lens.max()
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(lmax, op=dist.ReduceOp.MAX)
        self.s16 = int(int(lmax.item()) < 65536)
        self.row_words = 5 + ((mc + 1) // 2 if self.s16 else mc)
        self.rows = z(max(R, 1), self.row_words, dt=i32)
        self.g_res = z(max(Rt, 1), 4)
        # NVLink exchange of the route rows (no NCCL on the step's path): double-buffered
        # row buffers and a flag array [2 phases][world] per shard, mapped into every peer
        W = plan.world
        self.p2p = (W > 1 and dist.is_initialized() and dist.get_backend() == "nccl"
                    and os.environ.get("PYG_SHARD_NCCL", "0") != "1")
        self.seq = 0
        if self.p2p:
            self.rows_buf = [self.rows, z(max(R, 1), self.row_words, dt=i32)]
            self.flags = z(2 * W)
            wins2 = exchange_windows([t.data_ptr() for t in self.rows_buf + [self.flags]],
                                     export, import_)
            self.rows_of = [torch.tensor([wins2[k][b] for k in range(W)], dtype=i64,
                                         device=device) for b in (0, 1)]
            self.flag_of = [torch.tensor([wins2[k][2] + 8 * W * ph for k in range(W)],
                                         dtype=i64, device=device) for ph in (0, 1)]
        self.g_group = z(max(Rt, 1), dt=i32)
        self.g_staged = z(max(Rt, 1), mc, dt=i32)

    # ---------------------------------------------------------------- directory
    def build_directory(self):
        """All-gather every shard's L2 records and (re)build the replicated directory."""
        cap = int(_lib._lib.pyg_dir_export_cap(self.ctx.h))
        rec = torch.empty((cap, 5), dtype=torch.int64, device=self.dev)  # 40-byte records
        n = C.c_int64()
        check(_lib._lib.pyg_dir_export_dev(self.ctx.h, _ptr(rec), cap, C.byref(n)))
        nt = torch.tensor([n.value], dtype=torch.int64, device=self.dev)
        counts = allgather_cat(nt).cpu().tolist() if dist.is_initialized() else [n.value]
        allrec = allgather_var(rec, counts) if dist.is_initialized() else rec[:n.value]
        check(_lib._lib.pyg_dir_build_dev(self.ctx.h, _ptr(allrec), int(allrec.shape[0])))

    # ---------------------------------------------------------------- the step
    def step(self, now: float, speculative=True, release=True, mode=1, ev_hash=None,
             marks=None, prehashed=False, after_gather=None):
        """marks: optional list; (name, cuda event, host time) appended at phase ends.
        prehashed: the batch's boundary hashes are already in batch.hashes (K1 ran on another
        stream).  after_gather: called once the all-gather of the route rows is enqueued --
        from there on every rank has finished the previous step, so peers no longer read
        this rank's other input set (the next step's K1 may overwrite it)."""
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
        W = plan.world
        # 1-2: local hash + staged rows
        if not prehashed:
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
        # 3: all-gather compact route rows (also the barrier that frees last step's shared
        # buffers); every rank unpacks the whole burst's reservations, groups, staged rows
        mc = max(nodes.max_cand, 1)
        self.seq += 1
        if self.p2p:
            # pack into this step's row buffer, signal the peers, wait for all of them (every
            # shard has then finished the previous step), unpack their rows over NVLink
            par = self.seq % 2
            check(lib.pyg_shard_pack_dev(ctx.h, _ptr(b.res), _ptr(b.group), _ptr(self.staged),
                                         plan.R_local, mc, self.s16, _ptr(self.rows_buf[par])))
            check(lib.pyg_shard_signal_dev(ctx.h, _ptr(self.flag_of[0]), W, plan.rank, self.seq))
            check(lib.pyg_shard_wait_dev(ctx.h, _ptr(self.flags), W, self.seq))
            check(lib.pyg_shard_unpack_peer_dev(ctx.h, _ptr(self.rows_of[par]), W,
                                                _ptr(self.req_off_d), plan.R_total, mc, self.s16,
                                                _ptr(self.g_res), _ptr(self.g_group),
                                                _ptr(self.g_staged)))
        else:
            check(lib.pyg_shard_pack_dev(ctx.h, _ptr(b.res), _ptr(b.group), _ptr(self.staged),
                                         plan.R_local, mc, self.s16, _ptr(self.rows)))
            g_rows = (allgather_var(self.rows[:plan.R_local], self.req_counts)
                      if dist.is_initialized() else self.rows[:plan.R_local])
            check(lib.pyg_shard_unpack_dev(ctx.h, _ptr(g_rows), plan.R_total, mc, self.s16,
                                           _ptr(self.g_res), _ptr(self.g_group),
                                           _ptr(self.g_staged)))
        g_res, g_group, g_staged = self.g_res, self.g_group, self.g_staged
        if after_gather is not None:
            after_gather()
        mark("allgather")
        # 4: route the whole burst (identical on every rank)
        ns = nodes.struct()
        check(lib.pyg_route_batch_dev(ctx.h, mode, C.byref(ns), _ptr(g_res), plan.R_total,
                                      _ptr(g_group), nodes.n_groups, _ptr(nodes.cand_off),
                                      _ptr(nodes.cand), nodes.max_cand, _ptr(g_staged), 0.05,
                                      _ptr(self.decisions), _ptr(self.placed_off),
                                      _ptr(self.placed)))
        mark("route")
        # 5: requests placed on my replicas: plan, pull their tokens/hashes from the origins
        check(lib.pyg_shard_recv_plan_dev(ctx.h, plan.R_total, _ptr(self.decisions), _ptr(self.peers),
                                          W, _ptr(self.req_off_d), self.cap_req,
                                          _ptr(self.recv_gidx), _ptr(self.recv_count),
                                          _ptr(self.recv_toff), _ptr(self.recv_hoff),
                                          _ptr(self.recv_wf), _ptr(self.recv_role)))
        check(lib.pyg_shard_pull_dev(ctx.h, _ptr(self.peers), W, _ptr(self.req_off_d),
                                     _ptr(self.recv_gidx), _ptr(self.recv_count),
                                     _ptr(self.recv_toff), _ptr(self.recv_hoff), _ptr(self.r_tok),
                                     self.cap_tok, _ptr(self.r_hash), self.cap_hash))
        check(lib.pyg_shard_local_placed_dev(ctx.h, _ptr(self.placed_off), _ptr(self.placed),
                                             _ptr(self.recv_gidx), _ptr(self.recv_count),
                                             _ptr(self.p_off), _ptr(self.p_loc)))
        mark("dispatch")
        # 6: admission on the owner (bounded sizes; the real count lives on the device)
        check(lib.pyg_admit_shard_dev(ctx.h, _ptr(self.r_tok), _ptr(self.recv_toff),
                                      _ptr(self.recv_hoff), _ptr(self.r_hash), _ptr(self.recv_wf),
                                      _ptr(self.recv_role), self.cap_req, _ptr(self.p_off),
                                      _ptr(self.p_loc), now, int(bool(speculative)),
                                      _ptr(self.adm), _ptr(self.m3), _ptr(self.l2_list),
                                      self.cap_hash, _ptr(self.counts)))
        mark("admit")
        # 7: the L3 promotions in engine order: rank g's admissions follow every lower rank's
        # (global replica order), so it waits for their L3 erase lists, applies them to its
        # replica of the shared L3, resolves its own in order and publishes its list; then
        # every shard applies the remaining lists and every other shard's L2-directory clears
        def resolve():
            check(lib.pyg_shard_l3_resolve_dev(ctx.h, _ptr(self.r_tok), _ptr(self.recv_toff),
                                               _ptr(self.recv_hoff), _ptr(self.r_hash),
                                               self.cap_req, _ptr(self.p_off), _ptr(self.p_loc),
                                               _ptr(self.adm), _ptr(self.m3), _ptr(self.l3_list),
                                               self.cap_hash, self.cap_hash, _ptr(self.counts)))

        me = plan.rank
        if self.p2p:
            if me > 0:
                check(lib.pyg_shard_wait_dev(ctx.h, _ptr(self.flags[W:]), me, self.seq))
                check(lib.pyg_shard_apply_lists_range_dev(ctx.h, _ptr(self.peers), W, me, 0, me,
                                                          0))
            resolve()
            check(lib.pyg_shard_signal_dev(ctx.h, _ptr(self.flag_of[1]), W, me, self.seq))
            check(lib.pyg_shard_wait_dev(ctx.h, _ptr(self.flags[W:]), W, self.seq))
        else:
            for k in range(W):   # one stream barrier per rank's turn
                if k == me:
                    check(lib.pyg_shard_apply_lists_range_dev(ctx.h, _ptr(self.peers), W, me, 0,
                                                              me, 0))
                    resolve()
                barrier_on_stream(self.dev)
        check(lib.pyg_shard_apply_lists_range_dev(ctx.h, _ptr(self.peers), W, me, me, W, 1))
        mark("l2l3_lists")
        # 8: release on the owner; results of my requests from their owners
        if release:
            check(lib.pyg_release_batch_dev(ctx.h, _ptr(self.recv_toff), _ptr(self.recv_hoff),
                                            _ptr(self.r_hash), self.cap_req, _ptr(self.p_off),
                                            _ptr(self.p_loc), _ptr(self.adm)))
        check(lib.pyg_shard_results_dev(ctx.h, _ptr(self.peers), W, _ptr(self.rep_off_d),
                                        _ptr(self.decisions), plan.req_base, plan.R_local,
                                        _ptr(self.out_adm), _ptr(self.out_m3)))
        mark("release+return")
        return {"decisions": self.decisions[:plan.R_total], "placed_off": self.placed_off,
                "placed": self.placed, "admitted": self.out_adm[:plan.R_local],
                "match3": self.out_m3[:plan.R_local], "staged": self.staged[:plan.R_local],
                "recv_count": self.recv_count}


def decisions_host(dec: torch.Tensor) -> np.ndarray:
    return dec.cpu().numpy().view(DEC_DTYPE).reshape(-1)
