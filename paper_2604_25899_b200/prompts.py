"""Device prompt assembly (csrc/k_prompt.cu).

assemble_prompt (prompt.cpp:128-164) builds each prompt from a template: literal words
and references into earlier exchanges.  A B200 serving loop keeps those exchanges in HBM
(responses are decoded there, earlier prompts were assembled there), so per step the host
ships only segment descriptors (pool offset, length) plus genuinely new tokens (task
text, per-request salts, unique suffixes); pyg_assemble_dev gathers the prompts on device.

PromptPool lays out one device token pool for a trace: every distinct resident sequence
(a word table, an earlier exchange) once, then a fresh region rewritten every step.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check
from .workload import _signed, fnv1a_u64_vec


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class PromptPool:
    def __init__(self, trace, device="cuda", pinned=True):
        seg = trace.segments
        if seg is None:
            raise ValueError("trace has no prompt segments")
        kinds, keys = seg["kind"], seg["key"]
        start, length, fresh = seg["start"], seg["len"], seg["fresh"]
        S = len(kinds)
        R = trace.R
        # resident ranges: one per distinct (kind, key), long enough for every use
        need = {}
        for k in range(S):
            if not fresh[k]:
                kk = (kinds[k], keys[k])
                need[kk] = max(need.get(kk, 0), int(start[k] + length[k]))
        base = {}
        off = 0
        for kk, n in need.items():
            base[kk] = off
            off += n
        self.resident_tokens = off
        fresh_len = int(length[fresh].sum()) if S else 0
        self.fresh_tokens = fresh_len
        self.pool = torch.empty(max(off + fresh_len, 1), dtype=torch.int64, device=device)
        for (kind, key), n in need.items():
            b = base[(kind, key)]
            if kind == "w":
                tab = seg["word_tables"][key]
                self.pool[b:b + n] = torch.from_numpy(tab[:n]).to(device)
            else:
                idx = torch.arange(n, dtype=torch.int64, device=device)
                self.pool[b:b + n] = fnv1a_u64_vec(idx, torch.full_like(idx, _signed(key)))
        # segment descriptors (pool offset, length) in request order; fresh ones point into
        # the fresh region, filled from host memory every step
        src = np.zeros(S, np.int64)
        f_pos = off
        fresh_host = []
        for k in range(S):
            if fresh[k]:
                src[k] = f_pos
                f_pos += int(length[k])
                idx = torch.arange(int(start[k]), int(start[k] + length[k]), dtype=torch.int64)
                fresh_host.append(fnv1a_u64_vec(idx, torch.full_like(idx, _signed(keys[k]))))
            else:
                src[k] = base[(kinds[k], keys[k])] + int(start[k])
        segs = np.stack([src, length.astype(np.int64)], axis=1) if S else np.zeros((0, 2), np.int64)
        seg_off = np.zeros(R + 1, np.int64)
        np.cumsum(np.bincount(seg["req"], minlength=R), out=seg_off[1:])
        fh = torch.cat(fresh_host) if fresh_host else torch.zeros(0, dtype=torch.int64)

        def host(a):
            t = torch.as_tensor(a)
            return t.pin_memory() if pinned else t

        # per-step host inputs (pinned) and their device twins
        self.h_seg_off, self.h_segs, self.h_fresh = host(seg_off), host(segs), host(fh)
        self.d_seg_off = torch.empty_like(self.h_seg_off, device=device)
        self.d_segs = torch.empty_like(self.h_segs, device=device)
        self.R = R
        self.n_tokens = int(trace.tok_off[-1])
        self.device = device

    @property
    def h2d_bytes(self):
        return int(self.h_seg_off.numel() * 8 + self.h_segs.numel() * 8 + self.h_fresh.numel() * 8)

    def upload(self):
        """The step's host->device traffic: segment descriptors and the fresh tokens (written
        straight into the pool's fresh region)."""
        self.d_seg_off.copy_(self.h_seg_off, non_blocking=True)
        self.d_segs.copy_(self.h_segs, non_blocking=True)
        if self.fresh_tokens:
            self.pool[self.resident_tokens:self.resident_tokens + self.fresh_tokens].copy_(
                self.h_fresh, non_blocking=True)

    def assemble(self, ctx, tok_off: torch.Tensor, tokens: torch.Tensor):
        """pyg_assemble_dev into (tok_off [R+1], tokens [>= n_tokens])."""
        check(_lib._lib.pyg_assemble_dev(ctx.h, self.R, _p(self.d_seg_off), _p(self.d_segs),
                                         _p(self.pool), _p(tok_off), _p(tokens)))

    def assemble_hash(self, ctx, b):
        """pyg_assemble_hash_dev: prompts, hash offsets and boundary hashes of DeviceBatch b
        in one pass (K1 fused with the gather)."""
        check(_lib._lib.pyg_assemble_hash_dev(ctx.h, self.R, _p(self.d_seg_off),
                                              _p(self.d_segs), int(self.h_segs.shape[0]),
                                              _p(self.pool), self.n_tokens, _p(b.tok_off),
                                              _p(b.tokens), _p(b.hash_off), _p(b.hashes)))


class PipelinedSteps:
    """Step after step through the public API with a three-stage pipeline, so a step's
    host->device upload, its prompt assembly and its chain hashing (K1) all overlap earlier
    steps' device work:

      copy stream    upload(k+2) ............................ upload(k+3)
      prep stream       assemble+K1(k+1) ....................... assemble+K1(k+2)
      compute        step(k) [K2 | route, admit, release] ... step(k+1) ...
      d2h stream                                  results(k) ...

    * staging sets (3): a step's uploaded inputs -- segment descriptors, fresh tokens,
      request metadata.  upload(k) only waits for assembly(k-3) to have consumed its set.
    * batch sets (2): tokens, offsets, boundary hashes, metadata.  prep(k+1) starts at step
      k's `after_gather` point: for one GPU right after step k's K2 (so K2 keeps the whole
      GPU), for the sharded step once step k's route rows are all-gathered -- by then every
      rank has finished step k-1, so no peer still reads batch set (k+1) % 2 over NVLink.
    * assembly and K1 are one kernel (pyg_assemble_hash_dev: the gather's HBM traffic hides
      under the INT-bound hashing), run on the prep stream's own (replica-less) pyg_ctx with
      its grid capped below the SM count, leaving SMs to the step's latency-bound kernels.
    * results: the step's outputs are snapshotted on the compute stream (device copies)
      and copied to pinned host memory on their own stream.

    Every step still uploads its own inputs and copies its own results back.
    `run_step(batch, k, after_gather)` launches the device step for a DeviceBatch whose
    hashes are already computed, calls `after_gather()` at its safe point and returns the
    tensors to copy back."""

    STAGING = 3

    def __init__(self, ctx, trace, batch, device, run_step, pinned_meta, results_like,
                 second_batch=None, hash_ctas=None):
        from . import batch as PB
        from ._lib import Context
        self.PB, self.ctx, self.dev = PB, ctx, device
        p0 = PromptPool(trace, device=device)
        self.pools = [p0] + [_ShiftedFresh(p0) for _ in range(self.STAGING - 1)]
        self.batches = [batch, second_batch or clone_batch(batch)]
        self.meta = pinned_meta          # (res, group, wf, role) pinned host tensors
        self.st_meta = [[torch.empty(t.shape, dtype=t.dtype, device=device) for t in pinned_meta]
                        for _ in range(self.STAGING)]
        self.results = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in results_like]
                        for _ in range(2)]
        self.snap = [[torch.empty(t.shape, dtype=t.dtype, device=device) for t in results_like]
                     for _ in range(2)]
        self.copy = torch.cuda.Stream(device=device)
        self.prep = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self.compute = torch.cuda.current_stream(device)
        idx = device.index if isinstance(device, torch.device) and device.index is not None \
            else torch.cuda.current_device()
        self.prep_ctx = Context(0, [], [], ctx.B, device=idx)
        self.prep_ctx.set_stream(C.c_void_p(self.prep.cuda_stream))
        if hash_ctas is None:
            n_sm = torch.cuda.get_device_properties(idx).multi_processor_count
            hash_ctas = max(1, n_sm - 8)
        self.prep_ctx.set_hash_ctas(hash_ctas)
        E = torch.cuda.Event
        self.up = [E() for _ in range(self.STAGING)]
        self.consumed = [E() for _ in range(self.STAGING)]
        self.ready = [E() for _ in range(2)]
        self.snapped = [E() for _ in range(2)]
        self.fetched = [E() for _ in range(2)]
        self.run_step = run_step
        self.marks = None  # experiments: a list -> (stage, step, stream event) appended

    def _mark(self, name, k, stream):
        if self.marks is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            self.marks.append((name, k, e))

    def _upload(self, k):
        j = k % self.STAGING
        with torch.cuda.stream(self.copy):
            if k >= self.STAGING:
                self.copy.wait_event(self.consumed[j])
            self._mark("upload0", k, self.copy)
            self.pools[j].upload()
            for dst, src in zip(self.st_meta[j], self.meta):
                dst.copy_(src, non_blocking=True)
            self._mark("upload1", k, self.copy)
            self.up[j].record(self.copy)

    def _prepare(self, k):
        """assembly + metadata + hash offsets + K1 of step k into batch set k % 2 (prep
        stream, ordered after everything issued on the compute stream so far)."""
        j, b = k % self.STAGING, self.batches[k % 2]
        with torch.cuda.stream(self.prep):
            self.prep.wait_stream(self.compute)
            self.prep.wait_event(self.up[j])
            self._mark("prep0", k, self.prep)
            for dst, src in zip((b.res, b.group, b.wf, b.role), self.st_meta[j]):
                dst.copy_(src, non_blocking=True)
            # prompt assembly fused with K1: one pass over the pool
            self.pools[j].assemble_hash(self.prep_ctx, b)
            self.consumed[j].record(self.prep)
            self._mark("prep1", k, self.prep)
            self.ready[k % 2].record(self.prep)

    def run(self, steps, first_index=0):
        for k in range(min(steps, self.STAGING)):
            self._upload(k)
        self._prepare(0)
        for k in range(steps):
            s = k % 2
            self.compute.wait_event(self.ready[s])
            self._mark("step0", k, self.compute)
            self.PB.bind_current_stream(self.ctx)
            called = []

            def nxt(kk=k + 1):
                if not called and kk < steps:
                    self._prepare(kk)
                called.append(1)
            outs = self.run_step(self.batches[s], first_index + k, nxt)
            nxt()  # a run_step without a safe point: prepare after the whole step
            self._mark("step1", k, self.compute)
            if k >= 2:  # snapshot set s was read back two steps ago
                self.compute.wait_event(self.fetched[s])
            for dst, src in zip(self.snap[s], outs):
                dst.copy_(src, non_blocking=True)
            self.snapped[s].record(self.compute)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.snapped[s])
                for dst, src in zip(self.results[s], self.snap[s]):
                    dst.copy_(src, non_blocking=True)
                self.fetched[s].record(self.d2h)
                self._mark("d2h1", k, self.d2h)
            if k + self.STAGING < steps:
                self._upload(k + self.STAGING)
        self.compute.synchronize()
        self.d2h.synchronize()

    @property
    def h2d_bytes(self):
        return self.pools[0].h2d_bytes + sum(int(t.numel() * t.element_size()) for t in self.meta)

    @property
    def d2h_bytes(self):
        return sum(int(t.numel() * t.element_size()) for t in self.results[0])


def clone_batch(b):
    """A second DeviceBatch with its own buffers of the same shapes."""
    from . import batch as PB
    e = torch.empty_like
    return PB.DeviceBatch(b.R, e(b.tokens), e(b.tok_off), e(b.hash_off), e(b.hashes), e(b.res),
                          e(b.group), e(b.wf), e(b.role), b.n_hashes, b.n_tokens)


class _ShiftedFresh:
    """Second input set over the same pool: identical resident part, its own fresh region
    (appended to the pool) and its own segment-descriptor buffers."""

    def __init__(self, p0: PromptPool):
        self.p0 = p0
        self.R, self.fresh_tokens = p0.R, p0.fresh_tokens
        base = p0.pool.numel()
        grown = torch.empty(base + p0.fresh_tokens, dtype=torch.int64, device=p0.pool.device)
        grown[:base] = p0.pool
        p0.pool = grown
        self.pool_owner = p0
        shift = base - p0.resident_tokens
        segs = p0.h_segs.clone()
        fresh_mask = segs[:, 0] >= p0.resident_tokens
        segs[fresh_mask, 0] += shift
        self.h_seg_off, self.h_segs, self.h_fresh = p0.h_seg_off, segs.pin_memory(), p0.h_fresh
        self.d_seg_off = torch.empty_like(p0.d_seg_off)
        self.d_segs = torch.empty_like(p0.d_segs)
        self.fresh_base = base

    @property
    def h2d_bytes(self):
        return self.p0.h2d_bytes

    def upload(self):
        self.d_seg_off.copy_(self.h_seg_off, non_blocking=True)
        self.d_segs.copy_(self.h_segs, non_blocking=True)
        if self.fresh_tokens:
            self.pool_owner.pool[self.fresh_base:self.fresh_base + self.fresh_tokens].copy_(
                self.h_fresh, non_blocking=True)

    def assemble(self, ctx, tok_off, tokens):
        check(_lib._lib.pyg_assemble_dev(ctx.h, self.R, _p(self.d_seg_off), _p(self.d_segs),
                                         _p(self.pool_owner.pool), _p(tok_off), _p(tokens)))

    def assemble_hash(self, ctx, b):
        check(_lib._lib.pyg_assemble_hash_dev(ctx.h, self.R, _p(self.d_seg_off),
                                              _p(self.d_segs), int(self.h_segs.shape[0]),
                                              _p(self.pool_owner.pool), self.p0.n_tokens,
                                              _p(b.tok_off), _p(b.tokens), _p(b.hash_off),
                                              _p(b.hashes)))
