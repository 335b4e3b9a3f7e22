"""ctypes bindings for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with one interface:

* ``Restated(B)``  -- oracle/liboracle.so, the C restatement (any block size B).
* ``Reference(B)`` -- oracle/_ref/libpythia_ref{16,64}.so, the reference's own
  C++ sources compiled unmodified (B fixed at 16 or 64; present only where
  oracle/Makefile could see /root/reference, or where the built .so travelled).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

BLOCK_DTYPE = np.dtype([("id", "<u8"), ("hash", "<u8"), ("s", "<i8"), ("e", "<i8"),
                        ("wf", "<i4"), ("role", "<i4"), ("la", "<f8"), ("pin", "<i4"),
                        ("alive", "<i4")])
DEC_DTYPE = np.dtype([("target", "<i4"), ("tiebreak", "<i4"), ("headroom", "<i8"),
                      ("oom_bound", "<f8")])
RES_DTYPE = np.dtype([("prompt_len", "<i8"), ("upper", "<i8"), ("alpha", "<f8"),
                      ("tokens_generated", "<i8")])


class Decision(C.Structure):
    _fields_ = [("target", C.c_int32), ("tiebreak", C.c_int32), ("headroom", C.c_int64),
                ("oom_bound", C.c_double)]

    def as_tuple(self):
        return (self.target, self.tiebreak, self.headroom, self.oom_bound)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def build_restated():
    so = os.path.join(HERE, "liboracle.so")
    src = os.path.join(HERE, "pyg_oracle.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "restated"])
    return so


def reference_available(B: int) -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", f"libpythia_ref{B}.so"))


class _Backend:
    B: int

    def _sig(self, name, res, *args):
        f = getattr(self.lib, name)
        f.restype = res
        f.argtypes = list(args)
        return f


class Restated(_Backend):
    kind = "port"

    def __init__(self, B: int = 16):
        self.B = int(B)
        self.lib = C.CDLL(build_restated())
        vp, i64, i32, u64, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
        s = self._sig
        s("o_fnv1a_u64", u64, u64, u64)
        s("o_fnv1a_bytes", u64, C.c_char_p, i64, u64)
        s("o_chain_hashes", i64, vp, i64, i64, vp)
        s("o_cache_new", vp, i64, i64)
        s("o_cache_delete", None, vp)
        s("o_cache_clone", vp, vp)
        s("o_cache_set_off", None, vp, i32)
        s("o_add_decode_tokens", None, vp, i64)
        s("o_l1_occupancy", i64, vp)
        s("o_l3_new", vp)
        s("o_l3_delete", None, vp)
        s("o_l3_clone", vp, vp)
        s("o_registry_new", vp)
        s("o_registry_delete", None, vp)
        s("o_registry_update", None, vp, i32, u64)
        s("o_registry_drop", None, vp, i32)
        s("o_store_of", vp, vp, vp, i32)
        s("o_counter_of", vp, vp, vp, i32)
        s("o_lookup", None, vp, vp, vp, i64, i64, vp)
        s("o_matched_prefix", i64, vp, vp, i64, vp, i64, i64)
        s("o_insert_chain", None, vp, i32, vp, i64, i64, i32, i32, dbl, i32, i64)
        s("o_unpin_chain", None, vp, vp, i64, i64, i64)
        s("o_tier_put", u64, vp, u64, i64, i64, i32, i32, dbl, i32, vp)
        s("o_tier_erase", None, vp, u64)
        s("o_tier_dump", i64, vp, vp, i64)
        s("o_evict_for_space", C.c_int, vp, i32, i64, vp, C.c_int, vp, i64, vp, vp)
        s("o_on_request_complete", i64, vp, i32, u64, C.c_int, vp, i64)
        s("o_apply_completion", None, vp, i64, vp, vp, dbl)
        s("o_route", Decision, i32, vp, vp, vp, vp, vp, vp, dbl)
        s("o_route_least_outstanding", i32, i32, vp, vp)
        s("o_erase_chain_span", None, vp, vp, i64, i64, i64, i64)
        s("o_completion_policy", None, vp, i32, vp, vp, i32, u64, dbl)
        s("o_admit", C.c_int, vp, vp, vp, vp, C.c_int, vp, i64, i32, i32, dbl, i64, vp)

    # -- hashing
    def fnv1a_u64(self, v, h=1469598103934665603):
        return self.lib.o_fnv1a_u64(v, h)

    def fnv1a_str(self, s: str):
        b = s.encode()
        return self.lib.o_fnv1a_bytes(b, len(b), 1469598103934665603)

    def chain_hashes(self, tokens):
        t = _u64(tokens)
        out = np.zeros(max(1, (len(t) + self.B - 1) // self.B), np.uint64)
        k = self.lib.o_chain_hashes(_p(t), len(t), self.B, _p(out))
        return out[:k]

    # -- objects
    def new_cache(self, l1, l2):
        return self.lib.o_cache_new(l1, l2)

    def free_cache(self, c):
        self.lib.o_cache_delete(c)

    def clone_cache(self, c):
        return self.lib.o_cache_clone(c)

    def new_l3(self):
        return self.lib.o_l3_new()

    def free_l3(self, l):
        self.lib.o_l3_delete(l)

    def clone_l3(self, l):
        return self.lib.o_l3_clone(l)

    def new_registry(self):
        return self.lib.o_registry_new()

    def free_registry(self, r):
        self.lib.o_registry_delete(r)

    def reg_update(self, r, wf, mask):
        self.lib.o_registry_update(r, wf, mask)

    def reg_drop(self, r, wf):
        self.lib.o_registry_drop(r, wf)

    # -- cache ops
    def lookup(self, c, l3, tokens):
        t = _u64(tokens)
        out = np.zeros(3, np.int64)
        self.lib.o_lookup(c, l3, _p(t), len(t), self.B, _p(out))
        return tuple(int(x) for x in out)

    def matched_prefix(self, c, l3, tier, tokens):
        t = _u64(tokens)
        h = self.chain_hashes(t)
        st = self.lib.o_store_of(c, l3, tier)
        return self.lib.o_matched_prefix(st, _p(t), len(t), _p(h), len(h), self.B)

    def insert_chain(self, c, tier, tokens, upto, wf, role, now, pin):
        t = _u64(tokens)
        self.lib.o_insert_chain(c, tier, _p(t), len(t), upto, wf, role, now, pin, self.B)

    def unpin_chain(self, c, tokens, upto):
        t = _u64(tokens)
        self.lib.o_unpin_chain(c, _p(t), len(t), upto, self.B)

    def put(self, c, l3, tier, h, s, e, wf, role, now, pin):
        st = self.lib.o_store_of(c, l3, tier)
        ctr = self.lib.o_counter_of(c, l3, tier)
        return self.lib.o_tier_put(st, h, s, e, wf, role, now, pin, ctr)

    def erase(self, c, l3, tier, bid):
        self.lib.o_tier_erase(self.lib.o_store_of(c, l3, tier), bid)

    def dump(self, c, l3, tier):
        st = self.lib.o_store_of(c, l3, tier)
        n = self.lib.o_tier_dump(st, None, 0)
        out = np.zeros(n, BLOCK_DTYPE)
        self.lib.o_tier_dump(st, _p(out), n)
        return out

    def occupancy(self, c, l3, tier):
        d = self.dump(c, l3, tier)
        return int((d["e"] - d["s"]).sum())

    def add_decode(self, c, n):
        self.lib.o_add_decode_tokens(c, n)

    def l1_occupancy(self, c):
        return self.lib.o_l1_occupancy(c)

    def evict(self, c, tier, needed, reg, speculative):
        nf = C.c_int64()
        ft = C.c_int64()
        ok = self.lib.o_evict_for_space(c, tier, needed, reg, int(speculative), None, 0,
                                        C.byref(nf), C.byref(ft))
        return bool(ok), None, ft.value  # ids unavailable after the fact; see evict_ids

    def evict_ids(self, c, tier, needed, reg, speculative, cap=1 << 20):
        nf = C.c_int64()
        ft = C.c_int64()
        ids = np.zeros(cap, np.uint64)
        ok = self.lib.o_evict_for_space(c, tier, needed, reg, int(speculative), _p(ids), cap,
                                        C.byref(nf), C.byref(ft))
        return bool(ok), ids[: nf.value].copy(), ft.value

    def complete(self, c, l3, wf, future_mask, now, profiled=True):
        n = self.lib.o_on_request_complete(c, wf, future_mask, int(profiled), None, 0)
        acts = np.zeros(max(n, 1), np.dtype([("kind", "<i4"), ("tier", "<i4"), ("id", "<u8")]))
        self.lib.o_on_request_complete(c, wf, future_mask, int(profiled), _p(acts), n)
        self.lib.o_apply_completion(_p(acts), n, c, l3, now)
        return n

    def admit(self, c, l3_lookup, l3_live, reg, speculative, seq, wf, role, now):
        """cache side of start_prefill (engine.cpp:799-829); returns (admitted, (l1,l2,l3))"""
        t = _u64(seq)
        m = np.zeros(3, np.int64)
        ok = self.lib.o_admit(c, l3_lookup, l3_live, reg, int(speculative), _p(t), len(t), wf,
                              role, now, self.B, _p(m))
        return bool(ok), tuple(int(x) for x in m)

    def l3_dead_sweep(self, l3, wf, mask):
        # apply_completion_policy's L3 pass (engine.cpp:1074-1080) via the policy helper with
        # zero replicas
        self.lib.o_completion_policy(None, 0, l3, self._scratch_reg(), wf, mask, 0.0)

    def _scratch_reg(self):
        if not hasattr(self, "_sreg"):
            self._sreg = self.new_registry()
        return self._sreg

    def erase_chain_span(self, c, l3, tier, tokens, frm, to):
        t = _u64(tokens)
        self.lib.o_erase_chain_span(self.lib.o_store_of(c, l3, tier), _p(t), len(t), frm, to,
                                    self.B)

    def route(self, replica_id, kv_capacity, asg_off, asg, staged, req, eps):
        rid = np.ascontiguousarray(replica_id, np.int32)
        cap = np.ascontiguousarray(kv_capacity, np.int64)
        off = np.ascontiguousarray(asg_off, np.int64)
        a = np.ascontiguousarray(asg, RES_DTYPE) if len(asg) else np.zeros(1, RES_DTYPE)
        st = np.ascontiguousarray(staged, np.int64)
        r = np.ascontiguousarray(np.array([req], RES_DTYPE))
        return self.lib.o_route(len(rid), _p(rid), _p(cap), _p(off), _p(a), _p(st), _p(r),
                                eps).as_tuple()

    def route_least_outstanding(self, replica_id, asg_off):
        rid = np.ascontiguousarray(replica_id, np.int32)
        off = np.ascontiguousarray(asg_off, np.int64)
        return self.lib.o_route_least_outstanding(len(rid), _p(rid), _p(off))


class Reference(_Backend):
    """The reference's own implementation (unmodified sources + oracle/ref_shim.cpp)."""

    kind = "reference"

    def __init__(self, B: int = 16):
        self.B = int(B)
        path = os.path.join(HERE, "_ref", f"libpythia_ref{self.B}.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        vp, i64, i32, u64, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
        s = self._sig
        s("pref_block_tokens", i64)
        assert self.lib.pref_block_tokens() == self.B
        s("pref_fnv1a_str", u64, C.c_char_p, i64)
        s("pref_fnv1a_u64", u64, u64, u64)
        s("pref_response_token", u64, C.c_char_p, i64)
        s("pref_chain_hashes", i64, vp, i64, vp)
        s("pref_cache_new", vp, i64, i64)
        s("pref_cache_free", None, vp)
        s("pref_cache_clone", vp, vp)
        s("pref_l3_new", vp)
        s("pref_l3_free", None, vp)
        s("pref_l3_clone", vp, vp)
        s("pref_lookup", None, vp, vp, vp, i64, vp)
        s("pref_matched_prefix", i64, vp, vp, i32, vp, i64)
        s("pref_insert_chain", None, vp, i32, vp, i64, i64, i32, i32, dbl, i32)
        s("pref_unpin_chain", None, vp, vp, i64, i64)
        s("pref_tier_put", u64, vp, vp, i32, u64, i64, i64, i32, i32, dbl, i32)
        s("pref_tier_erase", None, vp, vp, i32, u64)
        s("pref_tier_occupancy", i64, vp, vp, i32)
        s("pref_tier_dump", i64, vp, vp, i32, vp, i64)
        s("pref_add_decode_tokens", None, vp, i64)
        s("pref_l1_occupancy", i64, vp)
        s("pref_registry_new", vp)
        s("pref_registry_free", None, vp)
        s("pref_registry_update", None, vp, i32, u64)
        s("pref_registry_drop", None, vp, i32)
        s("pref_evict", i32, vp, i32, i64, vp, i32, vp, i64, vp, vp)
        s("pref_route", Decision, i32, vp, vp, vp, vp, vp, vp, dbl)
        s("pref_route_least_outstanding", i32, i32, vp, vp)
        s("pref_future_mask", i64, C.c_char_p, C.c_char_p, vp)
        s("pref_expected_distance", i64, C.c_char_p, C.c_char_p, C.c_char_p, vp)
        s("pref_complete_mask", i64, vp, vp, i32, u64, dbl)
        s("pref_complete_expr", i64, vp, vp, i32, C.c_char_p, C.c_char_p, dbl)
        s("pref_l3_dead_sweep", None, vp, i32, u64)
        s("pref_erase_chain_span", None, vp, vp, i32, vp, i64, i64, i64)
        s("pref_step", i64, vp, i32, vp, vp, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
          vp, i32, dbl, dbl, i32, vp, vp)
        s("pref_burst", i64, vp, i32, vp, vp, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp,
          vp, vp, i32, dbl, dbl, i32, i32, vp, vp, vp, vp)
        s("pref_release", None, vp, vp, vp, i32, vp, vp)
        s("pref_assemble", i32, C.c_char_p, i32, C.c_char_p, vp, vp, vp, vp, i32, vp, i64, vp,
          vp)

    def fnv1a_u64(self, v, h=1469598103934665603):
        return self.lib.pref_fnv1a_u64(v, h)

    def fnv1a_str(self, s: str):
        b = s.encode()
        return self.lib.pref_fnv1a_str(b, len(b))

    def response_token(self, rid: str, i: int):
        return self.lib.pref_response_token(rid.encode(), i)

    def chain_hashes(self, tokens):
        t = _u64(tokens)
        out = np.zeros(max(1, (len(t) + self.B - 1) // self.B), np.uint64)
        k = self.lib.pref_chain_hashes(_p(t), len(t), _p(out))
        return out[:k]

    def new_cache(self, l1, l2):
        return self.lib.pref_cache_new(l1, l2)

    def free_cache(self, c):
        self.lib.pref_cache_free(c)

    def clone_cache(self, c):
        return self.lib.pref_cache_clone(c)

    def new_l3(self):
        return self.lib.pref_l3_new()

    def free_l3(self, l):
        self.lib.pref_l3_free(l)

    def clone_l3(self, l):
        return self.lib.pref_l3_clone(l)

    def new_registry(self):
        return self.lib.pref_registry_new()

    def free_registry(self, r):
        self.lib.pref_registry_free(r)

    def reg_update(self, r, wf, mask):
        self.lib.pref_registry_update(r, wf, mask)

    def reg_drop(self, r, wf):
        self.lib.pref_registry_drop(r, wf)

    def lookup(self, c, l3, tokens):
        t = _u64(tokens)
        out = np.zeros(3, np.int64)
        self.lib.pref_lookup(c, l3, _p(t), len(t), _p(out))
        return tuple(int(x) for x in out)

    def matched_prefix(self, c, l3, tier, tokens):
        t = _u64(tokens)
        return self.lib.pref_matched_prefix(c, l3, tier, _p(t), len(t))

    def insert_chain(self, c, tier, tokens, upto, wf, role, now, pin):
        t = _u64(tokens)
        self.lib.pref_insert_chain(c, tier, _p(t), len(t), upto, wf, role, now, pin)

    def unpin_chain(self, c, tokens, upto):
        t = _u64(tokens)
        self.lib.pref_unpin_chain(c, _p(t), len(t), upto)

    def put(self, c, l3, tier, h, s, e, wf, role, now, pin):
        return self.lib.pref_tier_put(c, l3, tier, h, s, e, wf, role, now, pin)

    def erase(self, c, l3, tier, bid):
        self.lib.pref_tier_erase(c, l3, tier, bid)

    def dump(self, c, l3, tier):
        n = self.lib.pref_tier_dump(c, l3, tier, None, 0)
        out = np.zeros(n, BLOCK_DTYPE)
        self.lib.pref_tier_dump(c, l3, tier, _p(out), n)
        return out

    def occupancy(self, c, l3, tier):
        return self.lib.pref_tier_occupancy(c, l3, tier)

    def add_decode(self, c, n):
        self.lib.pref_add_decode_tokens(c, n)

    def l1_occupancy(self, c):
        return self.lib.pref_l1_occupancy(c)

    def evict_ids(self, c, tier, needed, reg, speculative, cap=1 << 20):
        nf = C.c_int64()
        ft = C.c_int64()
        ids = np.zeros(cap, np.uint64)
        ok = self.lib.pref_evict(c, tier, needed, reg, int(speculative), _p(ids), cap,
                                 C.byref(nf), C.byref(ft))
        return bool(ok), ids[: nf.value].copy(), ft.value

    def complete(self, c, l3, wf, future_mask, now, profiled=True):
        if not profiled:
            return 0
        return self.lib.pref_complete_mask(c, l3, wf, future_mask, now)

    def complete_expr(self, c, l3, wf, expr, history, now):
        return self.lib.pref_complete_expr(c, l3, wf, expr.encode(), ",".join(history).encode(),
                                           now)

    def admit(self, c, l3_lookup, l3_live, reg, speculative, seq, wf, role, now):
        """start_prefill cache side (engine.cpp:799-829) composed from reference calls."""
        m = self.lookup(c, l3_lookup, seq)
        L = len(seq)
        ok, _, _ = self.evict_ids(c, 0, L - m[0], reg, speculative, cap=1)
        if not ok:
            return False, m
        reusable = max(m)
        l2_part = max(min(reusable, m[1]) - m[0], 0)
        l12 = max(m[0], m[1])
        l3_part = max(reusable - l12, 0)
        if l2_part > 0:
            self.erase_chain_span(c, None, 1, seq, m[0], m[0] + l2_part)
        if l3_part > 0:
            self.erase_chain_span(c, l3_live, 2, seq, l12, reusable)
        self.insert_chain(c, 0, seq, L, wf, role, now, +1)
        return True, m

    def step(self, caches, l3, reg, speculative, tokens, tok_off, res, group, wf, role, cl, mode,
             eps, now, release, want_out=True):
        """pref_step: one burst through the reference engine's call pattern (C++)."""
        R = len(tok_off) - 1
        arr = (C.c_void_p * len(caches))(*caches)
        t = _u64(tokens)
        off = np.ascontiguousarray(tok_off, np.int64)
        rs = np.ascontiguousarray(res, RES_DTYPE)
        g = np.ascontiguousarray(group, np.int32)
        w = np.ascontiguousarray(wf, np.int32)
        ro = np.ascontiguousarray(role, np.int32)
        a = np.ascontiguousarray(cl.asg, RES_DTYPE) if len(cl.asg) else np.zeros(1, RES_DTYPE)
        rid = np.ascontiguousarray(cl.replica_id, np.int32)
        kv = np.ascontiguousarray(cl.kv_capacity, np.int64)
        ao = np.ascontiguousarray(cl.asg_off, np.int64)
        co = np.ascontiguousarray(cl.cand_off, np.int32)
        cd = np.ascontiguousarray(cl.cand, np.int32)
        dec = np.zeros(max(R, 1), np.dtype([("target", "<i4"), ("tiebreak", "<i4"),
                                            ("headroom", "<i8"), ("oom_bound", "<f8")]))
        adm = np.zeros(max(R, 1), np.int32)
        n = self.lib.pref_step(C.cast(arr, C.c_void_p), len(caches), l3, reg, int(speculative),
                               _p(t), _p(off), R, _p(rs), _p(g), _p(w), _p(ro), _p(rid), _p(kv),
                               _p(ao), _p(a), _p(co), _p(cd), mode, eps, now, int(release),
                               _p(dec) if want_out else None, _p(adm) if want_out else None)
        return n, dec[:R], adm[:R]

    def burst(self, caches, l3, reg, speculative, tokens, tok_off, res, group, wf, role,
              replica_id, kv_capacity, asg_off, asg, cand_off, cand, eps, now, hash_once=True,
              threads=1, want_staged=False):
        """pref_burst: one burst of the steady-state bench through the reference's calls
        (node table given as a CSR; no release).  Returns (decisions, admitted, match3,
        staged or None)."""
        R = len(tok_off) - 1
        arr = (C.c_void_p * len(caches))(*caches)
        t = _u64(tokens)
        off = np.ascontiguousarray(tok_off, np.int64)
        rs = np.ascontiguousarray(res, RES_DTYPE)
        g = np.ascontiguousarray(group, np.int32)
        w = np.ascontiguousarray(wf, np.int32)
        ro = np.ascontiguousarray(role, np.int32)
        a = np.ascontiguousarray(asg, RES_DTYPE) if len(asg) else np.zeros(1, RES_DTYPE)
        rid = np.ascontiguousarray(replica_id, np.int32)
        kv = np.ascontiguousarray(kv_capacity, np.int64)
        ao = np.ascontiguousarray(asg_off, np.int64)
        co = np.ascontiguousarray(cand_off, np.int32)
        cd = np.ascontiguousarray(cand, np.int32)
        G = len(co) - 1
        mc = max(1, int(np.max(np.diff(co))) if G else 1)
        dec = np.zeros(max(R, 1), DEC_DTYPE)
        adm = np.zeros(max(R, 1), np.int32)
        m3 = np.zeros((max(R, 1), 3), np.int64)
        st = np.zeros((max(R, 1), mc), np.int32) if want_staged else None
        self.lib.pref_burst(C.cast(arr, C.c_void_p), len(caches), l3, reg, int(speculative),
                            _p(t), _p(off), R, _p(rs), _p(g), _p(w), _p(ro), _p(rid), _p(kv),
                            _p(ao), _p(a), _p(co), _p(cd), G, eps, now, int(bool(hash_once)),
                            int(threads), _p(dec), _p(adm), _p(m3),
                            _p(st) if st is not None else None)
        return dec[:R], adm[:R], m3[:R], (st[:R] if st is not None else None)

    def release(self, caches, tokens, tok_off, rep, admitted):
        """pref_release: unpin_chain of an earlier burst's admitted requests."""
        arr = (C.c_void_p * len(caches))(*caches)
        t = _u64(tokens)
        R = len(tok_off) - 1
        self.lib.pref_release(C.cast(arr, C.c_void_p), _p(t),
                              _p(np.ascontiguousarray(tok_off, np.int64)), R,
                              _p(np.ascontiguousarray(rep, np.int32)),
                              _p(np.ascontiguousarray(admitted, np.int32)))

    def assemble(self, text: str, exchanges: dict, prefix=False):
        """pref_assemble: (rc, tokens, complete) of assemble_prompt / assemble_resolvable_prefix
        (prompt.cpp:128-164) over a MapPromptHistory; rc 1 = nullopt, -1 = parse error."""
        ids = list(exchanges)
        req = [np.asarray(exchanges[k][0], np.uint64) for k in ids]
        resp = [np.asarray(exchanges[k][1], np.uint64) for k in ids]
        ro = np.zeros(len(ids) + 1, np.int64)
        np.cumsum([len(x) for x in req], out=ro[1:])
        so = np.zeros(len(ids) + 1, np.int64)
        np.cumsum([len(x) for x in resp], out=so[1:])
        rt = np.concatenate(req + [np.zeros(1, np.uint64)])
        st = np.concatenate(resp + [np.zeros(1, np.uint64)])
        cap = int(ro[-1] + so[-1]) + 64 * (len(text) + 1)
        out = np.zeros(cap, np.uint64)
        n = C.c_int64()
        comp = C.c_int32()
        rc = self.lib.pref_assemble(text.encode(), len(ids), "\n".join(ids).encode(), _p(ro),
                                    _p(rt), _p(so), _p(st), int(bool(prefix)), _p(out), cap,
                                    C.byref(n), C.byref(comp))
        return rc, (out[:n.value].copy() if rc == 0 else None), bool(comp.value)

    def future_mask(self, expr, history):
        m = C.c_uint64()
        rc = self.lib.pref_future_mask(expr.encode(), ",".join(history).encode(), C.byref(m))
        return None if rc < 0 else m.value

    def expected_distance(self, expr, history, role):
        d = C.c_double()
        rc = self.lib.pref_expected_distance(expr.encode(), ",".join(history).encode(),
                                             role.encode(), C.byref(d))
        if rc < 0:
            raise ValueError("history not locatable")
        return None if rc == 1 else d.value

    def l3_dead_sweep(self, l3, wf, mask):
        self.lib.pref_l3_dead_sweep(l3, wf, mask)

    def erase_chain_span(self, c, l3, tier, tokens, frm, to):
        t = _u64(tokens)
        self.lib.pref_erase_chain_span(c, l3, tier, _p(t), len(t), frm, to)

    def route(self, replica_id, kv_capacity, asg_off, asg, staged, req, eps):
        rid = np.ascontiguousarray(replica_id, np.int32)
        cap = np.ascontiguousarray(kv_capacity, np.int64)
        off = np.ascontiguousarray(asg_off, np.int64)
        a = np.ascontiguousarray(asg, RES_DTYPE) if len(asg) else np.zeros(1, RES_DTYPE)
        st = np.ascontiguousarray(staged, np.int64)
        r = np.ascontiguousarray(np.array([req], RES_DTYPE))
        return self.lib.pref_route(len(rid), _p(rid), _p(cap), _p(off), _p(a), _p(st), _p(r),
                                   eps).as_tuple()

    def route_least_outstanding(self, replica_id, asg_off):
        rid = np.ascontiguousarray(replica_id, np.int32)
        off = np.ascontiguousarray(asg_off, np.int64)
        return self.lib.pref_route_least_outstanding(len(rid), _p(rid), _p(off))
