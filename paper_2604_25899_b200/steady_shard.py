"""The steady-state burst step over the GPUs of one box, one process per GPU.

Rank g of W owns whole models: global replicas [g N/W, (g+1) N/W) of an N-replica cluster
whose models are contiguous replica blocks (config 4: 8 models x 32), their L1/L2 tiers and
node-table entries; the shared L3 and the L2 directory are replicated.  Every rank brings
its own burst of R requests per step (weak scaling); burst k of the job is the
concatenation of the ranks' bursts in rank order (global issue order).  Step k on rank g:

  1. releases: its replicas' admitted requests of burst k-1 with hold 1 and of burst k-2
     with hold 2 (unpin_chain on the owner, hierarchy.cpp:132-142)
  2. registry updates of the whole burst k (replicated FutureRegistry, engine.cpp:605-609)
  3. K2: staged row of its own requests against all candidates (replicated directory)
  4. route rows of every rank over NVLink (flag barrier, peer reads)
  5. K3: sequential-commit route of the requests of ITS models only, against its own node
     table (base + burst k-1's held placements) -- a model's requests only ever see that
     model's replicas (engine.cpp:630-638), so a model's commit order is independent of
     the others and K3 splits by model owner with no further exchange
  6. owner pulls its placed requests' tokens / hashes from their origins over NVLink,
     admits them (K4/K5), L3 promotions in engine order chained over the ranks, L2/L3
     erase lists applied everywhere (shard.py)
  7. node table of burst k+1: base + burst k's placements with hold 2 (owner-local)
Only the route rows, the pulled requests and the erase lists cross NVLink; no host
synchronisation inside the step.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import batch as PB
from . import steady as S
from ._lib import check
from .shard import ShardedStep, ShardPlan, allgather_cat


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def owned_groups(cl, rep_lo, rep_hi):
    """Groups (models) whose candidates all lie in [rep_lo, rep_hi)."""
    G = len(cl.cand_off) - 1
    own = []
    for g in range(G):
        c = cl.cand[cl.cand_off[g]:cl.cand_off[g + 1]]
        if len(c) and c.min() >= rep_lo and c.max() < rep_hi:
            own.append(g)
        elif len(c) and (c.min() < rep_hi and c.max() >= rep_lo):
            raise ValueError(f"model {g} straddles ranks: replicas must split by model")
    return own


class SteadyShardStep(ShardedStep):
    """ShardedStep of one burst in the steady sequence (its own IPC window, receive lists and
    flags).  route_nodes: this rank's node table (global replica ids, own models'
    candidates only)."""

    def step_steady(self, now, route_nodes, after_gather=None, ev=None, after_staged=None):
        """ev: optional dict name -> CUDA event, recorded at the phase ends (experiments)."""
        ctx, plan, b, nodes = self.ctx, self.plan, self.b, self.nodes
        lib = _lib._lib
        W = plan.world

        def mark(name):
            if ev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev[name] = e
        PB.bind_current_stream(ctx)
        mark("start")
        check(lib.pyg_staged_matrix_dev(ctx.h, _ptr(b.tokens), _ptr(b.tok_off), _ptr(b.hash_off),
                                        _ptr(b.hashes), plan.R_local, _ptr(b.group),
                                        nodes.n_groups, _ptr(nodes.cand_off), _ptr(nodes.cand),
                                        nodes.max_cand, _ptr(self.staged)))
        if after_staged is not None:
            after_staged()
        mark("staged")
        mc = max(nodes.max_cand, 1)
        self.seq += 1
        if self.p2p:
            par = self.seq % 2
            check(lib.pyg_shard_pack_dev(ctx.h, _ptr(b.res), _ptr(b.group), _ptr(self.staged),
                                         plan.R_local, mc, self.s16, _ptr(self.rows_buf[par])))
            check(lib.pyg_shard_signal_dev(ctx.h, _ptr(self.flag_of[0]), W, plan.rank, self.seq))
            check(lib.pyg_shard_wait_dev(ctx.h, _ptr(self.flags), W, self.seq))
            check(lib.pyg_shard_unpack_peer_own_dev(ctx.h, _ptr(self.rows_of[par]), W,
                                                    _ptr(self.req_off_d), plan.R_total, mc,
                                                    self.s16, self.own_mask, _ptr(self.g_res),
                                                    _ptr(self.g_group), _ptr(self.g_staged)))
        else:
            from .shard import allgather_var
            check(lib.pyg_shard_pack_dev(ctx.h, _ptr(b.res), _ptr(b.group), _ptr(self.staged),
                                         plan.R_local, mc, self.s16, _ptr(self.rows)))
            g_rows = (allgather_var(self.rows[:plan.R_local], self.req_counts)
                      if dist.is_initialized() else self.rows[:plan.R_local])
            check(lib.pyg_shard_unpack_dev(ctx.h, _ptr(g_rows), plan.R_total, mc, self.s16,
                                           _ptr(self.g_res), _ptr(self.g_group),
                                           _ptr(self.g_staged)))
        mark("exchange")
        if after_gather is not None:
            after_gather()
        # K3 over this rank's models only (other models' requests have no local candidates)
        ns = route_nodes.struct()
        check(lib.pyg_route_batch_dev(ctx.h, 1, C.byref(ns), _ptr(self.g_res), plan.R_total,
                                      _ptr(self.g_group), route_nodes.n_groups,
                                      _ptr(route_nodes.cand_off), _ptr(route_nodes.cand),
                                      route_nodes.max_cand, _ptr(self.g_staged), 0.05,
                                      _ptr(self.decisions), _ptr(self.placed_off),
                                      _ptr(self.placed)))
        mark("route")
        check(lib.pyg_shard_recv_plan_dev(ctx.h, plan.R_total, _ptr(self.decisions),
                                          _ptr(self.peers), W, _ptr(self.req_off_d), self.cap_req,
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
        check(lib.pyg_admit_shard_dev(ctx.h, _ptr(self.r_tok), _ptr(self.recv_toff),
                                      _ptr(self.recv_hoff), _ptr(self.r_hash), _ptr(self.recv_wf),
                                      _ptr(self.recv_role), self.cap_req, _ptr(self.p_off),
                                      _ptr(self.p_loc), now, 1, _ptr(self.adm), _ptr(self.m3),
                                      _ptr(self.l2_list), self.cap_hash, _ptr(self.counts)))
        mark("pull+admit")
        me = plan.rank

        def resolve():
            check(lib.pyg_shard_l3_resolve_dev(ctx.h, _ptr(self.r_tok), _ptr(self.recv_toff),
                                               _ptr(self.recv_hoff), _ptr(self.r_hash),
                                               self.cap_req, _ptr(self.p_off), _ptr(self.p_loc),
                                               _ptr(self.adm), _ptr(self.m3), _ptr(self.l3_list),
                                               self.cap_hash, self.cap_hash, _ptr(self.counts)))
        if self.p2p:
            # the lower ranks' L3 lists matter only if an admission here matched in L3: the
            # wait + apply run on the device only then (a rank without L3 matches publishes
            # its empty list at once, so the chain serializes only the ranks that need it)
            check(lib.pyg_shard_l3_prepare_dev(ctx.h, _ptr(self.peers), _ptr(self.flags[W:]), W,
                                               me, self.seq))
            resolve()
            check(lib.pyg_shard_signal_dev(ctx.h, _ptr(self.flag_of[1]), W, me, self.seq))
            check(lib.pyg_shard_wait_dev(ctx.h, _ptr(self.flags[W:]), W, self.seq))
        else:
            from .shard import barrier_on_stream
            for k in range(W):
                if k == me:
                    check(lib.pyg_shard_apply_lists_range_dev(ctx.h, _ptr(self.peers), W, me, 0,
                                                              me, 0))
                    resolve()
                barrier_on_stream(self.dev)
        mark("l3_chain")
        # every rank's L3 erasures (re-applying the lower ranks' is a no-op) + the L2 clears
        check(lib.pyg_shard_apply_lists_range_dev(ctx.h, _ptr(self.peers), W, me, 0, W, 1))
        mark("lists")

    def release_hold(self, hold_all, h):
        """Unpin this burst's admitted requests of hold h on this rank's replicas."""
        check(_lib._lib.pyg_release_hold_dev(self.ctx.h, _ptr(self.recv_toff),
                                             _ptr(self.recv_hoff), _ptr(self.r_hash),
                                             self.cap_req, _ptr(self.p_off), _ptr(self.p_loc),
                                             _ptr(self.adm), _ptr(hold_all), h,
                                             _ptr(self.recv_gidx)))


class ShardedSteady:
    """Rank `rank` of `world`: its ctx (own replicas), its bursts (steady.Burst list, burst
    k = global sub-burst k*world + rank) and the per-burst exchange windows."""

    def __init__(self, ctx, cl, rank, world, bursts, B, device):
        self.ctx, self.cl, self.rank, self.world, self.dev = ctx, cl, rank, world, device
        n = cl.n_replicas
        if n % world:
            raise ValueError("replicas must split evenly over the GPUs")
        per = n // world
        self.rep_lo, self.rep_hi = rank * per, (rank + 1) * per
        self.own = owned_groups(cl, self.rep_lo, self.rep_hi)
        R = bursts[0].R
        self.R = R
        self.plan = ShardPlan([per] * world, [R] * world, rank, B)
        self.nodes = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg,
                                     cl.cand_off, cl.cand, device=device)  # K2: every group
        # K3: own groups' candidates only; the node table (global ids) carried across bursts
        G = len(cl.cand_off) - 1
        co = np.zeros(G + 1, np.int32)
        cand = []
        for g in range(G):
            c = cl.cand[cl.cand_off[g]:cl.cand_off[g + 1]] if g in self.own else []
            cand.extend(int(x) for x in c)
            co[g + 1] = len(cand)
        self.route_nodes = PB.upload_nodes(cl.replica_id, cl.kv_capacity, cl.asg_off, cl.asg, co,
                                           np.asarray(cand, np.int32), device=device)
        self.base_off, self.base = self.route_nodes.asg_off, self.route_nodes.asg
        A = int(cl.asg_off[-1])
        Rt = R * world
        self.route_nodes.asg_off = torch.zeros_like(self.base_off)
        self.route_nodes.asg = torch.zeros((A + Rt + 1, 4), dtype=torch.int64, device=device)
        kv_loc = cl.kv_capacity[self.rep_lo:self.rep_hi]
        tt = int(sum(b.b.n_tokens for b in bursts[:1])) * world
        self.bursts = bursts
        self.steps = [SteadyShardStep(ctx, self.plan, b.b, self.nodes, device, kv_loc, tt)
                      for b in bursts]
        own_mask = 0
        if max(self.own, default=0) < 64:
            for g in self.own:
                own_mask |= 1 << g
        for st in self.steps:
            st.own_mask = own_mask if own_mask else 0
        # per burst: hold of every global request, and the registry pairs of the whole burst
        self.hold_all, self.reg = [], []
        for k, b in enumerate(bursts):
            h = np.concatenate([S.hold_of(k * world + g, R, R) for g in range(world)])
            self.hold_all.append(torch.from_numpy(h).to(device))
            wf = allgather_cat(b.b.wf[:R].contiguous()).cpu().numpy()
            role = allgather_cat(b.b.role[:R].contiguous()).cpu().numpy()
            rw, rm = S.registry_pairs(wf, role)
            self.reg.append((torch.from_numpy(rw).to(device),
                             torch.from_numpy(rm.view(np.int64)).to(device), len(rw),
                             int(wf.max()) if len(wf) else 0))

    def reserve(self):
        """Size the device registry for every burst's workflows (replicated registry)."""
        self.ctx.registry_reserve(max(r[3] for r in self.reg))

    def build_directory(self):
        self.steps[0].build_directory()

    def compose_nodes(self, k):
        """node table of burst k: base + burst k-1's placements still held (hold 2)."""
        if k >= 1:
            st = self.steps[k - 1]
            po, pl, req, hold = st.placed_off, st.placed, st.g_res, self.hold_all[k - 1]
        else:
            po = pl = req = hold = None
        check(_lib._lib.pyg_nodes_compose_dev(
            self.ctx.h, self.cl.n_replicas, _ptr(self.base_off), _ptr(self.base), _ptr(po),
            _ptr(pl), _ptr(req), _ptr(hold), 2, _ptr(self.route_nodes.asg_off),
            _ptr(self.route_nodes.asg)))

    def step(self, k, now, after_gather=None, ev=None, after_staged=None):
        """Everything of step k after K1 of this rank's burst k."""
        PB.bind_current_stream(self.ctx)
        if ev is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ev["begin"] = e
        for h in (1, 2):
            if k - h >= 0:
                self.steps[k - h].release_hold(self.hold_all[k - h], h)
        self.compose_nodes(k)
        rw, rm, nr, mx = self.reg[k]
        check(_lib._lib.pyg_registry_update_batch_dev(self.ctx.h, nr, _ptr(rw), _ptr(rm), mx))
        self.steps[k].step_steady(now, self.route_nodes, after_gather, ev, after_staged)
        return self.steps[k]
