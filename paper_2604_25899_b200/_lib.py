"""ctypes binding of libpyg_b200.so (the C-ABI in include/pyg.h).

The shared library is the only compute path: if it is missing this module
raises at import time (there is no CPU fallback).  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` or
``python paper_2604_25899_b200/build.py``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PYG_SO: experiments only (A/B of two builds on one box)
SO_PATH = os.environ.get("PYG_SO") or os.path.join(HERE, "libpyg_b200.so")

if not os.path.exists(SO_PATH):
    raise ImportError(f"{SO_PATH} is not built; run paper_2604_25899_b200/build.py "
                      "(the B200 path has no CPU fallback)")

_lib = C.CDLL(SO_PATH)

vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double

BLOCK_DTYPE = np.dtype([("id", "<u8"), ("hash", "<u8"), ("s", "<i8"), ("e", "<i8"),
                        ("wf", "<i4"), ("role", "<i4"), ("la", "<f8"), ("pin", "<i4"),
                        ("alive", "<i4")])
RES_DTYPE = np.dtype([("prompt_len", "<i8"), ("upper", "<i8"), ("alpha", "<f8"),
                      ("tokens_generated", "<i8")])
DEC_DTYPE = np.dtype([("target", "<i4"), ("tiebreak", "<i4"), ("headroom", "<i8"),
                      ("oom_bound", "<f8")])

PYG_ERRORS = {-1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ECAPACITY", -5: "ENOTSUP"}


class PygError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"pyg error {PYG_ERRORS.get(code, code)}: {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [("block_tokens", i32), ("n_replicas", i32), ("device", i32), ("reserved", i32),
                ("l1_capacity", vp), ("l2_capacity", vp), ("min_blocks", i64)]


class Block(C.Structure):
    _fields_ = [("block_id", u64), ("chain_hash", u64), ("span_start", i64), ("span_end", i64),
                ("workflow", i32), ("role", i32), ("last_access", dbl), ("pin_count", i32),
                ("alive", i32)]


class Reservation(C.Structure):
    _fields_ = [("prompt_len", i64), ("upper", i64), ("alpha", dbl), ("tokens_generated", i64)]


class Decision(C.Structure):
    _fields_ = [("target", i32), ("tiebreak", i32), ("headroom", i64), ("oom_bound", dbl)]


class NodesDev(C.Structure):
    _fields_ = [("replica_id", vp), ("kv_capacity", vp), ("asg_off", vp), ("asg", vp)]


def _sig(name, *args, res=C.c_int):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("pyg_create", C.POINTER(Config), C.POINTER(vp))
_sig("pyg_destroy", vp, res=None)
_sig("pyg_last_error", res=C.c_char_p)
_sig("pyg_set_stream", vp, vp)
_sig("pyg_set_hash_ctas", vp, i32)
_sig("pyg_synchronize", vp)
_sig("pyg_kernel_launches", vp, res=i64)
_sig("pyg_set_capacity", vp, i32, i64, i64)
_sig("pyg_assemble_dev", vp, i32, vp, vp, vp, vp, vp)
_sig("pyg_assemble_hash_dev", vp, i32, vp, vp, i64, vp, i64, vp, vp, vp, vp)
_sig("pyg_form_batch_dev", vp, i32, vp, vp, vp, vp, dbl, dbl, vp, vp)
_sig("pyg_preemption_victim_dev", vp, i32, vp, vp, dbl, dbl, vp)
_sig("pyg_stage_plan_dev", vp, vp, vp, vp, vp, i32, vp, i32, vp, vp, i32, vp, vp, vp)
_sig("pyg_chain_hashes", vp, vp, i64, vp, vp)
_sig("pyg_tier_put", vp, i32, i32, u64, i64, i64, i32, i32, dbl, i32, vp)
_sig("pyg_tier_erase", vp, i32, i32, u64)
_sig("pyg_tier_find", vp, i32, i32, u64, vp, vp)
_sig("pyg_tier_stats", vp, i32, i32, vp, vp, vp)
_sig("pyg_tier_dump", vp, i32, i32, vp, i64, vp)
_sig("pyg_matched_prefix", vp, i32, i32, vp, i64, vp)
_sig("pyg_lookup", vp, i32, vp, i64, i32, vp)
_sig("pyg_insert_chain", vp, i32, i32, vp, i64, i64, i32, i32, dbl, i32)
_sig("pyg_unpin_chain", vp, i32, vp, i64, i64)
_sig("pyg_add_decode_tokens", vp, i32, i64)
_sig("pyg_l1_occupancy", vp, i32, vp)
_sig("pyg_erase_chain_span", vp, i32, i32, vp, i64, i64, i64)
_sig("pyg_set_replica_off", vp, i32, i32)
_sig("pyg_registry_update", vp, i32, u64)
_sig("pyg_registry_drop", vp, i32)
_sig("pyg_evict_for_space", vp, i32, i32, i64, i32, vp, i64, vp, vp, vp)
_sig("pyg_complete", vp, i32, i32, u64, i32, dbl, vp)
_sig("pyg_l3_dead_sweep", vp, i32, u64)
_sig("pyg_completion_policy", vp, i32, u64, dbl)
_sig("pyg_route", vp, i32, vp, vp, vp, vp, vp, vp, dbl, vp)
_sig("pyg_route_least_outstanding", vp, i32, vp, vp, vp)
_sig("pyg_check_device_error", vp)
# batched (device pointers)
_sig("pyg_hash_offsets_dev", vp, vp, i32, vp, vp)
_sig("pyg_hash_batch_dev", vp, vp, vp, i32, vp, vp)
_sig("pyg_staged_matrix_dev", vp, vp, vp, vp, vp, i32, vp, i32, vp, vp, i32, vp)
_sig("pyg_set_shard", vp, i32, i32)
_sig("pyg_dir_export_cap", vp, res=i64)
_sig("pyg_dir_export_dev", vp, vp, i64, vp)
_sig("pyg_dir_build_dev", vp, vp, i64)
_sig("pyg_admit_shard_dev", vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, dbl, i32, vp, vp, vp, i64, vp)
_sig("pyg_shard_l3_resolve_dev", vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, i64, i64, vp)
_sig("pyg_dir_clear_dev", vp, vp, i64, vp)
_sig("pyg_l3_erase_hashes_dev", vp, vp, i64, vp)
_sig("pyg_gather_csr_dev", vp, vp, vp, vp, i64, vp, vp)
_sig("pyg_ipc_export", vp, vp, vp)
_sig("pyg_next_use_dev", vp, vp, i32, vp, i32, vp, vp, vp, i32, vp, vp)
_sig("pyg_block_next_use_dev", vp, i32, i32, vp, i32, vp, i32, vp, i64, vp)
_sig("pyg_registry_from_cursors_dev", vp, i32, i32, vp, vp, vp, vp)
_sig("pyg_ipc_import", vp, vp, i64, vp)
_sig("pyg_shard_recv_plan_dev", vp, i32, vp, vp, i32, vp, i64, vp, vp, vp, vp, vp, vp)
_sig("pyg_shard_unpack_peer_dev", vp, vp, i32, vp, i32, i32, i32, vp, vp, vp)
_sig("pyg_shard_unpack_peer_own_dev", vp, vp, i32, vp, i32, i32, i32, C.c_uint64, vp, vp, vp)
_sig("pyg_shard_signal_dev", vp, vp, i32, i32, i64)
_sig("pyg_shard_wait_dev", vp, vp, i32, i64)
_sig("pyg_shard_pack_dev", vp, vp, vp, vp, i32, i32, i32, vp)
_sig("pyg_shard_unpack_dev", vp, vp, i32, i32, i32, vp, vp, vp)
_sig("pyg_shard_pull_dev", vp, vp, i32, vp, vp, vp, vp, vp, vp, i64, vp, i64)
_sig("pyg_shard_local_placed_dev", vp, vp, vp, vp, vp, vp, vp)
_sig("pyg_stats", vp, vp, i32)
_sig("pyg_lookup_all", vp, vp, i64, i32, i32, vp)
_sig("pyg_set_hash_split", vp, i64)
_sig("pyg_set_hash_grid", vp, i32)
_sig("pyg_set_hash_gate", vp, vp)
_sig("pyg_set_hash_memo", vp, i32)
_sig("pyg_nodes_compose_dev", vp, i32, vp, vp, vp, vp, vp, vp, i32, vp, vp)
_sig("pyg_release_hold_dev", vp, vp, vp, vp, i32, vp, vp, vp, vp, i32, vp)
_sig("pyg_registry_update_batch_dev", vp, i32, vp, vp, i32)
_sig("pyg_registry_reserve", vp, i32)
_sig("pyg_shard_apply_lists_dev", vp, vp, i32, i32)
_sig("pyg_shard_apply_lists_range_dev", vp, vp, i32, i32, i32, i32, i32)
_sig("pyg_shard_l3_prepare_dev", vp, vp, vp, i32, i32, i64)
_sig("pyg_shard_results_dev", vp, vp, i32, vp, vp, i64, i32, vp, vp)
_sig("pyg_lookup_batch_dev", vp, vp, vp, vp, vp, i32, vp, i32, vp)
_sig("pyg_route_batch_dev", vp, i32, C.POINTER(NodesDev), vp, i32, vp, i32, vp, vp, i32, vp,
     dbl, vp, vp, vp)
_sig("pyg_admit_batch_dev", vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, dbl, i32, vp, vp)
_sig("pyg_release_batch_dev", vp, vp, vp, vp, i32, vp, vp, vp)



class BatchHost(C.Structure):
    _fields_ = [("n_req", i32), ("reserved", i32), ("tokens", vp), ("tok_off", vp), ("req", vp),
                ("group", vp), ("workflow", vp), ("role", vp)]


class NodesHost(C.Structure):
    _fields_ = [("replica_id", vp), ("kv_capacity", vp), ("asg_off", vp), ("asg", vp),
                ("n_groups", i32), ("reserved", i32), ("cand_off", vp), ("cand", vp)]


_sig("pyg_step_host", vp, C.POINTER(BatchHost), C.POINTER(NodesHost), i32, dbl, dbl, i32, i32,
     vp, vp, vp)

EXPORTED = [n for n in dir(_lib) if n.startswith("pyg_")]


def last_error() -> str:
    m = _lib.pyg_last_error()
    return m.decode() if m else ""


def check(rc):
    if rc != 0:
        raise PygError(rc, last_error())
    return rc


def _p(a):
    return None if a is None else a.ctypes.data_as(vp)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


class Context:
    """One GPU's share of the cluster: n_replicas CacheHierarchy instances (L1+L2) and the
    shared L3 store, all resident in HBM."""

    def __init__(self, n_replicas, l1_capacity, l2_capacity, block_tokens=16, device=0,
                 min_blocks=0):
        l1 = np.ascontiguousarray(np.broadcast_to(np.asarray(l1_capacity, np.int64),
                                                  (n_replicas,)))
        l2 = np.ascontiguousarray(np.broadcast_to(np.asarray(l2_capacity, np.int64),
                                                  (n_replicas,)))
        self.B = int(block_tokens)
        self.n_replicas = int(n_replicas)
        cfg = Config(self.B, self.n_replicas, int(device), 0, _p(l1), _p(l2), int(min_blocks))
        h = vp()
        check(_lib.pyg_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self._l1, self._l2 = l1, l2

    def close(self):
        if getattr(self, "h", None):
            _lib.pyg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing
    def set_stream(self, stream_ptr):
        check(_lib.pyg_set_stream(self.h, stream_ptr))

    def set_hash_ctas(self, n):
        check(_lib.pyg_set_hash_ctas(self.h, int(n)))

    def synchronize(self):
        check(_lib.pyg_synchronize(self.h))

    def kernel_launches(self) -> int:
        return _lib.pyg_kernel_launches(self.h)

    def check_device_error(self):
        check(_lib.pyg_check_device_error(self.h))

    def registry_reserve(self, max_wf: int):
        check(_lib.pyg_registry_reserve(self.h, int(max_wf)))

    def set_hash_grid(self, mode: str):
        """K1 grid: "persistent" (default), "tasks" (one task per warp), "tasks1" (one task
        per warp, at most one K1 CTA per SM)."""
        check(_lib.pyg_set_hash_grid(self.h, {"tasks": 0, "persistent": 1, "tasks1": 2}[mode]))

    def set_hash_memo(self, on: bool):
        """K1 prefix memo (default off; see pyg.h)."""
        check(_lib.pyg_set_hash_memo(self.h, int(bool(on))))

    def set_hash_gate(self, step_ctx):
        """K1 of this ctx pauses while step_ctx runs an admission (None: no gate)."""
        check(_lib.pyg_set_hash_gate(self.h, step_ctx.h if step_ctx is not None else None))

    def set_hash_split(self, min_tokens: int):
        check(_lib.pyg_set_hash_split(self.h, int(min_tokens)))

    def counters(self, reset=False) -> dict:
        """pyg_stats: eviction / admission counters (synchronizes the ctx stream)."""
        out = np.zeros(8, np.int64)
        check(_lib.pyg_stats(self.h, out.ctypes.data, int(bool(reset))))
        return {"evicted_blocks": int(out[0]), "evicted_tokens": int(out[1]),
                "evictions": int(out[2]), "unsatisfied": int(out[3]),
                "admissions": int(out[4]), "admitted": int(out[5]),
                "l3_promoted_tokens": int(out[6])}

    # -- hashing
    def chain_hashes(self, tokens):
        t = _u64(tokens)
        out = np.zeros(max(1, (len(t) + self.B - 1) // self.B), np.uint64)
        n = C.c_int64()
        check(_lib.pyg_chain_hashes(self.h, _p(t), len(t), _p(out), C.byref(n)))
        return out[: n.value]

    # -- TierStore level (tier 2 == shared L3)
    def put(self, replica, tier, h, s, e, wf, role, now, pin):
        out = C.c_uint64()
        check(_lib.pyg_tier_put(self.h, replica, tier, h, s, e, wf, role, now, pin,
                                C.byref(out)))
        return out.value

    def erase(self, replica, tier, bid):
        check(_lib.pyg_tier_erase(self.h, replica, tier, bid))

    def find(self, replica, tier, h):
        b = Block()
        f = C.c_int32()
        check(_lib.pyg_tier_find(self.h, replica, tier, h, C.byref(b), C.byref(f)))
        return b if f.value else None

    def stats(self, replica, tier):
        occ, cap, nb = C.c_int64(), C.c_int64(), C.c_int64()
        check(_lib.pyg_tier_stats(self.h, replica, tier, C.byref(occ), C.byref(cap),
                                  C.byref(nb)))
        return occ.value, cap.value, nb.value

    def dump(self, replica, tier):
        n = C.c_int64()
        check(_lib.pyg_tier_dump(self.h, replica, tier, None, 0, C.byref(n)))
        out = np.zeros(n.value, BLOCK_DTYPE)
        check(_lib.pyg_tier_dump(self.h, replica, tier, _p(out), n.value, C.byref(n)))
        return out

    def matched_prefix(self, replica, tier, tokens):
        t = _u64(tokens)
        out = C.c_int64()
        check(_lib.pyg_matched_prefix(self.h, replica, tier, _p(t), len(t), C.byref(out)))
        return out.value

    # -- CacheHierarchy level
    def lookup_all(self, tokens, with_l3=True, n_rep=None):
        """pyg_lookup_all: (l1, l2, l3) of one prompt on replicas 0..n_rep-1."""
        t = np.ascontiguousarray(tokens, np.uint64)
        n = self.n_replicas if n_rep is None else int(n_rep)
        out = np.zeros((max(n, 1), 3), np.int64)
        check(_lib.pyg_lookup_all(self.h, t.ctypes.data, len(t), int(bool(with_l3)), n,
                                  out.ctypes.data))
        return out[:n]

    def lookup(self, replica, tokens, with_l3=True):
        t = _u64(tokens)
        out = np.zeros(3, np.int64)
        check(_lib.pyg_lookup(self.h, replica, _p(t), len(t), int(bool(with_l3)), _p(out)))
        return tuple(int(x) for x in out)

    def insert_chain(self, replica, tier, tokens, upto, wf, role, now, pin):
        t = _u64(tokens)
        check(_lib.pyg_insert_chain(self.h, replica, tier, _p(t), len(t), upto, wf, role, now,
                                    pin))

    def unpin_chain(self, replica, tokens, upto):
        t = _u64(tokens)
        check(_lib.pyg_unpin_chain(self.h, replica, _p(t), len(t), upto))

    def add_decode_tokens(self, replica, n):
        check(_lib.pyg_add_decode_tokens(self.h, replica, n))

    def l1_occupancy(self, replica):
        out = C.c_int64()
        check(_lib.pyg_l1_occupancy(self.h, replica, C.byref(out)))
        return out.value

    def erase_chain_span(self, replica, tier, tokens, frm, to):
        t = _u64(tokens)
        check(_lib.pyg_erase_chain_span(self.h, replica, tier, _p(t), len(t), frm, to))

    def set_replica_off(self, replica, off=True):
        check(_lib.pyg_set_replica_off(self.h, replica, int(bool(off))))

    # -- manager
    def registry_update(self, wf, mask):
        check(_lib.pyg_registry_update(self.h, wf, mask))

    def registry_drop(self, wf):
        check(_lib.pyg_registry_drop(self.h, wf))

    def evict_for_space(self, replica, tier, needed, speculative, cap=1 << 20):
        ids = np.zeros(max(cap, 1), np.uint64)
        nf, ft, sat = C.c_int64(), C.c_int64(), C.c_int32()
        check(_lib.pyg_evict_for_space(self.h, replica, tier, needed, int(bool(speculative)),
                                       _p(ids), cap, C.byref(nf), C.byref(ft), C.byref(sat)))
        return bool(sat.value), ids[: min(nf.value, cap)].copy(), ft.value

    def complete(self, replica, wf, future_mask, now, profiled=True):
        n = C.c_int64()
        check(_lib.pyg_complete(self.h, replica, wf, future_mask, int(bool(profiled)), now,
                                C.byref(n)))
        return n.value

    def l3_dead_sweep(self, wf, mask):
        check(_lib.pyg_l3_dead_sweep(self.h, wf, mask))

    def completion_policy(self, wf, mask, now):
        check(_lib.pyg_completion_policy(self.h, wf, mask, now))

    # -- router
    def route(self, replica_id, kv_capacity, asg_off, asg, staged, req, eps):
        rid = np.ascontiguousarray(replica_id, np.int32)
        cap = np.ascontiguousarray(kv_capacity, np.int64)
        off = np.ascontiguousarray(asg_off, np.int64)
        a = np.ascontiguousarray(asg, RES_DTYPE) if len(asg) else np.zeros(1, RES_DTYPE)
        st = np.ascontiguousarray(staged, np.int64)
        r = Reservation(*[x.item() if hasattr(x, "item") else x for x in req])
        d = Decision()
        check(_lib.pyg_route(self.h, len(rid), _p(rid), _p(cap), _p(off), _p(a), _p(st),
                             C.byref(r), eps, C.byref(d)))
        return (d.target, d.tiebreak, d.headroom, d.oom_bound)

    def route_least_outstanding(self, replica_id, asg_off):
        rid = np.ascontiguousarray(replica_id, np.int32)
        off = np.ascontiguousarray(asg_off, np.int64)
        out = C.c_int32()
        check(_lib.pyg_route_least_outstanding(self.h, len(rid), _p(rid), _p(off),
                                               C.byref(out)))
        return out.value
