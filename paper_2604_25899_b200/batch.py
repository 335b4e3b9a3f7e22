"""Device-resident batched hot path (the throughput path).

A *step* routes one batch of R requests through the cluster shard held by a
``Context``, exactly as the reference engine composes the hot-path calls
(SURVEY.md CS-1 + CS-2 restricted to the batch):

  1. K1  hash every prompt                 chain_boundary_hashes   hierarchy.cpp:21-30
  2. K2  staged matrix (L2 prefix per      node_view               engine.cpp:640-648
         request x candidate replica)
  3. K3  route every request               sched::route            router.cpp:19-50
         (SEQ_COMMIT: engine order, each placement committed before the next
          request, engine.cpp:650-692; SNAPSHOT: all against one frozen state)
  4. K4/K5 admit placed requests per       start_prefill           engine.cpp:799-829
         replica in placement order: lookup(seq,&l3) -> evict_for_space(L1)
         -> erase promoted L2 span -> insert_chain(L1, pin+1); promoted L3 spans
         are erased after all admissions (erasures commute)
  5. K5  optional release: unpin_chain of admitted requests (completion without
         response; keeps the cluster in steady state between bench steps)

Buffers are torch CUDA tensors (plumbing); all compute is libpyg_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import DEC_DTYPE, RES_DTYPE, check

SNAPSHOT = 0
SEQ_COMMIT = 1


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _i64_view(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.int64)


@dataclass
class DeviceBatch:
    R: int
    tokens: torch.Tensor      # int64 view of uint64 tokens
    tok_off: torch.Tensor     # int64 [R+1]
    hash_off: torch.Tensor    # int64 [R+1]
    hashes: torch.Tensor      # int64 view of uint64 boundary hashes
    res: torch.Tensor         # int64 [R, 4] (pyg_reservation; alpha as double bits)
    group: torch.Tensor       # int32 [R]
    wf: torch.Tensor          # int32 [R]
    role: torch.Tensor        # int32 [R]
    n_hashes: int
    n_tokens: int


@dataclass
class DeviceNodes:
    replica_id: torch.Tensor  # int32 [n_rep]
    kv_capacity: torch.Tensor # int64 [n_rep]
    asg_off: torch.Tensor     # int64 [n_rep+1]
    asg: torch.Tensor         # int64 [A, 4]
    cand_off: torch.Tensor    # int32 [G+1]
    cand: torch.Tensor        # int32 [sum]
    n_groups: int
    max_cand: int

    def struct(self):
        return _lib.NodesDev(self.replica_id.data_ptr(), self.kv_capacity.data_ptr(),
                             self.asg_off.data_ptr(), self.asg.data_ptr())


def upload_batch(ctx: _lib.Context, tokens: np.ndarray, tok_off: np.ndarray, res: np.ndarray,
                 group: np.ndarray, wf: np.ndarray, role: np.ndarray,
                 device="cuda") -> DeviceBatch:
    R = len(tok_off) - 1
    t_tok = torch.from_numpy(_i64_view(np.asarray(tokens, np.uint64))).to(device)
    t_off = torch.from_numpy(np.ascontiguousarray(tok_off, np.int64)).to(device)
    nb = (np.diff(np.asarray(tok_off, np.int64)) + ctx.B - 1) // ctx.B
    hoff = np.zeros(R + 1, np.int64)
    np.cumsum(nb, out=hoff[1:])
    t_hoff = torch.from_numpy(hoff).to(device)
    t_hash = torch.empty(max(int(hoff[-1]), 1), dtype=torch.int64, device=device)
    r = np.ascontiguousarray(res, RES_DTYPE)
    t_res = torch.from_numpy(r.view(np.int64).reshape(R, 4).copy()).to(device)
    return DeviceBatch(R, t_tok, t_off, t_hoff, t_hash, t_res,
                       torch.from_numpy(np.ascontiguousarray(group, np.int32)).to(device),
                       torch.from_numpy(np.ascontiguousarray(wf, np.int32)).to(device),
                       torch.from_numpy(np.ascontiguousarray(role, np.int32)).to(device),
                       int(hoff[-1]), int(tok_off[-1]))


def upload_nodes(replica_id, kv_capacity, asg_off, asg, cand_off, cand, device="cuda"):
    a = np.ascontiguousarray(asg, RES_DTYPE) if len(asg) else np.zeros(1, RES_DTYPE)
    co = np.asarray(cand_off, np.int32)
    return DeviceNodes(
        torch.from_numpy(np.ascontiguousarray(replica_id, np.int32)).to(device),
        torch.from_numpy(np.ascontiguousarray(kv_capacity, np.int64)).to(device),
        torch.from_numpy(np.ascontiguousarray(asg_off, np.int64)).to(device),
        torch.from_numpy(a.view(np.int64).reshape(-1, 4).copy()).to(device),
        torch.from_numpy(co.copy()).to(device),
        torch.from_numpy(np.ascontiguousarray(cand, np.int32)).to(device),
        len(co) - 1, int(np.max(np.diff(co))) if len(co) > 1 else 0)


@dataclass
class StepOut:
    decisions: torch.Tensor   # int64 [R, 3] (pyg_decision)
    staged: torch.Tensor      # int32 [R, max_cand]
    placed_off: torch.Tensor  # int32 [n_rep+1]
    placed: torch.Tensor      # int32 [R]
    admitted: torch.Tensor    # int32 [R]
    match3: torch.Tensor      # int64 [R, 3]

    def host(self):
        d = self.decisions.cpu().numpy().view(DEC_DTYPE).reshape(-1)
        return {"decisions": d, "staged": self.staged.cpu().numpy(),
                "placed_off": self.placed_off.cpu().numpy(), "placed": self.placed.cpu().numpy(),
                "admitted": self.admitted.cpu().numpy(), "match3": self.match3.cpu().numpy()}


def alloc_out(ctx: _lib.Context, b: DeviceBatch, nodes: DeviceNodes, device="cuda") -> StepOut:
    R = b.R
    return StepOut(torch.zeros((max(R, 1), 3), dtype=torch.int64, device=device),
                   torch.zeros((max(R, 1), max(nodes.max_cand, 1)), dtype=torch.int32,
                               device=device),
                   torch.zeros(ctx.n_replicas + 1, dtype=torch.int32, device=device),
                   torch.zeros(max(R, 1), dtype=torch.int32, device=device),
                   torch.zeros(max(R, 1), dtype=torch.int32, device=device),
                   torch.zeros((max(R, 1), 3), dtype=torch.int64, device=device))


def bind_current_stream(ctx):
    """Launch the library's kernels on torch's current stream (orders them after the
    torch copies that fill the batch buffers)."""
    ctx.set_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream))


def hash_batch(ctx, b: DeviceBatch):
    check(_lib._lib.pyg_hash_batch_dev(ctx.h, _ptr(b.tokens), _ptr(b.tok_off), b.R,
                                       _ptr(b.hash_off), _ptr(b.hashes)))


def staged_matrix(ctx, b: DeviceBatch, nodes: DeviceNodes, out: StepOut):
    check(_lib._lib.pyg_staged_matrix_dev(ctx.h, _ptr(b.tokens), _ptr(b.tok_off),
                                          _ptr(b.hash_off), _ptr(b.hashes), b.R, _ptr(b.group),
                                          nodes.n_groups, _ptr(nodes.cand_off), _ptr(nodes.cand),
                                          nodes.max_cand, _ptr(out.staged)))


def route_batch(ctx, b: DeviceBatch, nodes: DeviceNodes, out: StepOut, mode=SEQ_COMMIT,
                eps=0.05):
    ns = nodes.struct()
    check(_lib._lib.pyg_route_batch_dev(ctx.h, mode, C.byref(ns), _ptr(b.res), b.R,
                                        _ptr(b.group), nodes.n_groups, _ptr(nodes.cand_off),
                                        _ptr(nodes.cand), nodes.max_cand, _ptr(out.staged), eps,
                                        _ptr(out.decisions), _ptr(out.placed_off),
                                        _ptr(out.placed)))


def admit_batch(ctx, b: DeviceBatch, out: StepOut, now: float, speculative=True):
    check(_lib._lib.pyg_admit_batch_dev(ctx.h, _ptr(b.tokens), _ptr(b.tok_off), _ptr(b.hash_off),
                                        _ptr(b.hashes), _ptr(b.wf), _ptr(b.role), b.R,
                                        _ptr(out.placed_off), _ptr(out.placed), now,
                                        int(bool(speculative)), _ptr(out.admitted),
                                        _ptr(out.match3)))


def release_batch(ctx, b: DeviceBatch, out: StepOut):
    check(_lib._lib.pyg_release_batch_dev(ctx.h, _ptr(b.tok_off), _ptr(b.hash_off),
                                          _ptr(b.hashes), b.R, _ptr(out.placed_off),
                                          _ptr(out.placed), _ptr(out.admitted)))


def lookup_batch(ctx, b: DeviceBatch, replica: torch.Tensor, with_l3=True):
    out = torch.zeros((max(b.R, 1), 3), dtype=torch.int64, device=b.tokens.device)
    check(_lib._lib.pyg_lookup_batch_dev(ctx.h, _ptr(b.tokens), _ptr(b.tok_off), _ptr(b.hash_off),
                                         _ptr(b.hashes), b.R, _ptr(replica), int(bool(with_l3)),
                                         _ptr(out)))
    return out


def step(ctx, b: DeviceBatch, nodes: DeviceNodes, out: StepOut, now: float, mode=SEQ_COMMIT,
         eps=0.05, speculative=True, release=True):
    """One routed-request pass over the batch (all device work, no host sync)."""
    bind_current_stream(ctx)
    hash_batch(ctx, b)
    staged_matrix(ctx, b, nodes, out)
    route_batch(ctx, b, nodes, out, mode, eps)
    admit_batch(ctx, b, out, now, speculative)
    if release:
        release_batch(ctx, b, out)
    return out


class HostStep:
    """The host-buffer batch entry (pyg_step_host): pinned host arrays in/out, every step
    copies the batch to the device, runs K1..K5 and copies the results back."""

    def __init__(self, ctx, tokens: np.ndarray, tok_off, res, group, wf, role, cluster,
                 pinned=True):
        def pin(a, dtype):
            a = np.ascontiguousarray(a, dtype)
            if not pinned or a.size == 0:
                return a
            t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
            v = t.numpy().view(dtype).reshape(a.shape)
            v[...] = a
            self._keep.append(t)
            return v

        self._keep = []
        self.ctx = ctx
        self.R = len(tok_off) - 1
        self.tokens = pin(tokens, np.uint64)
        self.tok_off = pin(tok_off, np.int64)
        self.res = pin(res, RES_DTYPE)
        self.group = pin(group, np.int32)
        self.wf = pin(wf, np.int32)
        self.role = pin(role, np.int32)
        cl = cluster
        self.rid = np.ascontiguousarray(cl.replica_id, np.int32)
        self.kv = np.ascontiguousarray(cl.kv_capacity, np.int64)
        self.aoff = np.ascontiguousarray(cl.asg_off, np.int64)
        self.asg = np.ascontiguousarray(cl.asg, RES_DTYPE) if len(cl.asg) else np.zeros(1, RES_DTYPE)
        self.coff = np.ascontiguousarray(cl.cand_off, np.int32)
        self.cand = np.ascontiguousarray(cl.cand, np.int32)
        self.out_dec = pin(np.zeros(max(self.R, 1), DEC_DTYPE), DEC_DTYPE)
        self.out_adm = pin(np.zeros(max(self.R, 1), np.int32), np.int32)
        self.out_m3 = pin(np.zeros((max(self.R, 1), 3), np.int64), np.int64)
        p = lambda a: a.ctypes.data  # noqa: E731
        self.bh = _lib.BatchHost(self.R, 0, p(self.tokens), p(self.tok_off), p(self.res),
                                 p(self.group), p(self.wf), p(self.role))
        self.nh = _lib.NodesHost(p(self.rid), p(self.kv), p(self.aoff), p(self.asg),
                                 len(self.coff) - 1, 0, p(self.coff), p(self.cand))

    @property
    def h2d_bytes(self):
        return int(self.tokens.nbytes + self.tok_off.nbytes + self.res.nbytes + self.group.nbytes
                   + self.wf.nbytes + self.role.nbytes + self.rid.nbytes + self.kv.nbytes
                   + self.aoff.nbytes + self.asg.nbytes + self.coff.nbytes + self.cand.nbytes)

    @property
    def d2h_bytes(self):
        return int(self.R * (DEC_DTYPE.itemsize + 4 + 24))

    def __call__(self, now, mode=SEQ_COMMIT, eps=0.05, speculative=True, release=True):
        check(_lib._lib.pyg_step_host(self.ctx.h, C.byref(self.bh), C.byref(self.nh), mode, eps,
                                      now, int(bool(speculative)), int(bool(release)),
                                      self.out_dec.ctypes.data, self.out_adm.ctypes.data,
                                      self.out_m3.ctypes.data))
        return self.out_dec, self.out_adm, self.out_m3
