"""Adapter giving the GPU Context the same interface as oracle.py_oracle backends,
so one scenario script drives the oracle and the CUDA path identically."""
import numpy as np


class _Proxy:
    def __init__(self, ctx):
        self.ctx = ctx


class Gpu:
    kind = "gpu"

    def __init__(self, B=16):
        from paper_2604_25899_b200 import Context
        self.B = B
        self._Context = Context
        self._last = None
        self._default = None

    def _ctx(self):
        if self._last is None:
            self._default = self._default or self._Context(1, 1 << 40, 1 << 40, self.B)
            return self._default
        return self._last

    def new_cache(self, l1, l2):
        self._last = self._Context(1, l1, l2, self.B)
        return _Proxy(self._last)

    def free_cache(self, c):
        c.ctx.close()

    def new_l3(self):
        return _Proxy(self._ctx())

    def free_l3(self, l):
        pass

    def new_registry(self):
        r = _Proxy(None)
        r.state = {}
        return r

    def free_registry(self, r):
        pass

    def reg_update(self, r, wf, mask):
        r.state[wf] = mask

    def reg_drop(self, r, wf):
        r.state[wf] = None

    @staticmethod
    def _sync_registry(ctx, r):
        for wf, m in r.state.items():
            if m is None:
                ctx.registry_drop(wf)
            else:
                ctx.registry_update(wf, m)

    def fnv1a_u64(self, v, h=1469598103934665603):
        raise NotImplementedError

    def chain_hashes(self, tokens):
        return self._ctx().chain_hashes(tokens)

    def lookup(self, c, l3, tokens):
        return c.ctx.lookup(0, tokens, with_l3=l3 is not None)

    def matched_prefix(self, c, l3, tier, tokens):
        return c.ctx.matched_prefix(0, tier, tokens)

    def insert_chain(self, c, tier, tokens, upto, wf, role, now, pin):
        c.ctx.insert_chain(0, tier, tokens, upto, wf, role, now, pin)

    def unpin_chain(self, c, tokens, upto):
        c.ctx.unpin_chain(0, tokens, upto)

    def put(self, c, l3, tier, h, s, e, wf, role, now, pin):
        t = tier if (tier != 2 or l3 is not None) else 1
        return c.ctx.put(0, t, h, s, e, wf, role, now, pin)

    def erase(self, c, l3, tier, bid):
        t = tier if (tier != 2 or l3 is not None) else 1
        c.ctx.erase(0, t, bid)

    def dump(self, c, l3, tier):
        t = tier if (tier != 2 or l3 is not None) else 1
        return c.ctx.dump(0, t)

    def occupancy(self, c, l3, tier):
        t = tier if (tier != 2 or l3 is not None) else 1
        return c.ctx.stats(0, t)[0]

    def add_decode(self, c, n):
        c.ctx.add_decode_tokens(0, n)

    def l1_occupancy(self, c):
        return c.ctx.l1_occupancy(0)

    def evict_ids(self, c, tier, needed, reg, speculative, cap=1 << 20):
        self._sync_registry(c.ctx, reg)
        return c.ctx.evict_for_space(0, tier, needed, speculative, cap)

    def complete(self, c, l3, wf, future_mask, now, profiled=True):
        return c.ctx.complete(0, wf, future_mask, now, profiled)

    def l3_dead_sweep(self, l3, wf, mask):
        l3.ctx.l3_dead_sweep(wf, mask)

    def erase_chain_span(self, c, l3, tier, tokens, frm, to):
        t = tier if (tier != 2 or l3 is not None) else 1
        c.ctx.erase_chain_span(0, t, tokens, frm, to)

    def route(self, replica_id, kv_capacity, asg_off, asg, staged, req, eps):
        return self._ctx().route(replica_id, kv_capacity, asg_off, asg, staged, req, eps)

    def route_least_outstanding(self, replica_id, asg_off):
        return self._ctx().route_least_outstanding(replica_id, asg_off)
