"""Synthetic agent-workflow traces built with the reference's token conventions.

Token content (so a trace hashes exactly as the reference engine's would):
  literal word w         -> fnv1a(w)                            tokens.hpp:22-28, prompt.cpp:11-21
  response token i of r  -> fnv1a(i, fnv1a("resp", fnv1a(r)))   tokens.hpp:42-44
  task token k of wf w   -> fnv1a(k, fnv1a("task", fnv1a(w)))   engine.cpp:570-574
  salt token k of req r  -> fnv1a(k, fnv1a(r, fnv1a("salt")))   engine.cpp:576-579
Prompt assembly follows rule_for (engine.cpp:348-379): role system-prompt
words ("sys_<role>_<i>", engine.cpp:339-346) + the carried prefix of the
previous stage's response + task tokens on stage 0 + sibling salt.

Every indexed token is fnv1a(index, H) for a per-segment key H, so a whole
trace is two gathers and one vectorized FNV pass (torch; CUDA when available).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

FNV_OFFSET = 1469598103934665603
FNV_PRIME = 1099511628211
M64 = (1 << 64) - 1
RES_DTYPE = np.dtype([("prompt_len", "<i8"), ("upper", "<i8"), ("alpha", "<f8"),
                      ("tokens_generated", "<i8")])
ALPHA = 1 - 0.99          # profiler/store.cpp:20 with confidence 0.99
GLOBAL_MAX_OUTPUT = 16384  # sim/config.hpp:95


def fnv1a_str(s: str, h: int = FNV_OFFSET) -> int:
    for c in s.encode():
        h = ((h ^ c) * FNV_PRIME) & M64
    return h


def fnv1a_u64(v: int, h: int = FNV_OFFSET) -> int:
    for i in range(8):
        h = ((h ^ ((v >> (8 * i)) & 0xFF)) * FNV_PRIME) & M64
    return h


def _signed(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


def fnv1a_u64_vec(v: torch.Tensor, h: torch.Tensor) -> torch.Tensor:
    """fnv1a(uint64 v, h) elementwise on int64 tensors (two's-complement wraparound)."""
    prime = torch.tensor(FNV_PRIME, dtype=torch.int64, device=v.device)
    for i in range(8):
        h = torch.bitwise_xor(h, torch.bitwise_and(torch.bitwise_right_shift(v, 8 * i), 0xFF))
        h = h * prime
    return h


def response_key(rid: str) -> int:
    return fnv1a_str("resp", fnv1a_str(rid))


def task_key(wid: str) -> int:
    return fnv1a_str("task", fnv1a_str(wid))


def salt_key(rid: str) -> int:
    return fnv1a_str(rid, fnv1a_str("salt"))


@dataclass
class Role:
    name: str
    model: int
    sys_tokens: int
    carry_tokens: int
    out_mean: float
    out_cv: float


@dataclass
class Trace:
    """Token CSR + per-request routing inputs, in issue order."""
    tokens: torch.Tensor          # int64 view of uint64 tokens (device of generation)
    tok_off: np.ndarray           # int64 [R+1]
    res: np.ndarray               # RES_DTYPE [R]
    group: np.ndarray             # int32 [R] model index == candidate group
    wf: np.ndarray                # int32 [R]
    role: np.ndarray              # int32 [R]
    roles: list = field(default_factory=list)
    n_models: int = 1
    name: str = ""
    segments: dict = None         # prompt segments (see _Builder.segments), for prompts.py

    @property
    def R(self):
        return len(self.tok_off) - 1

    @property
    def n_tokens(self):
        return int(self.tok_off[-1])

    def tokens_np(self) -> np.ndarray:
        return self.tokens.cpu().numpy().view(np.uint64)

    def prompt(self, r) -> np.ndarray:
        t = self.tokens[int(self.tok_off[r]):int(self.tok_off[r + 1])]
        return t.cpu().numpy().view(np.uint64)

    def subset(self, idx) -> "Trace":
        idx = np.asarray(idx)
        lens = np.diff(self.tok_off)[idx]
        off = np.zeros(len(idx) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        parts = [self.tokens[int(self.tok_off[r]):int(self.tok_off[r + 1])] for r in idx]
        toks = torch.cat(parts) if parts else self.tokens[:0]
        return Trace(toks, off, self.res[idx].copy(), self.group[idx].copy(), self.wf[idx].copy(),
                     self.role[idx].copy(), self.roles, self.n_models, self.name + "[subset]")


def _p99(mean, cv):
    s2 = math.log(1 + cv * cv)
    mu = math.log(mean) - s2 / 2
    return int(min(GLOBAL_MAX_OUTPUT, max(1, round(math.exp(mu + 2.3263478740408408 * math.sqrt(s2))))))


def _lognormal(rng, mean, cv, size):
    s2 = math.log(1 + cv * cv)
    mu = math.log(mean) - s2 / 2
    return np.clip(np.rint(rng.lognormal(mu, math.sqrt(s2), size)), 1, GLOBAL_MAX_OUTPUT).astype(np.int64)


def _with_segments(b, tr):
    tr.segments = b.segments()
    return tr


class _Builder:
    """Accumulates segment descriptors; materializes all tokens in one vectorized pass."""

    def __init__(self):
        self.word_tables = {}
        self.seg_req, self.seg_kind, self.seg_key, self.seg_start, self.seg_len = [], [], [], [], []
        self.seg_fresh = []

    def words(self, prefix, n):
        key = (prefix, n)
        if key not in self.word_tables:
            self.word_tables[key] = np.array([_signed(fnv1a_str(f"{prefix}_{i}")) for i in range(n)],
                                             np.int64)
        return key

    def add(self, r, kind, key, start, length, fresh=False):
        """One prompt segment.  fresh: new content of this request (task text, salt, unique
        suffix) that a serving system must upload; otherwise it is history already resident
        on the device (sys-prompt words, an earlier exchange's tokens)."""
        if length <= 0:
            return
        self.seg_req.append(r)
        self.seg_kind.append(kind)
        self.seg_key.append(key)
        self.seg_start.append(start)
        self.seg_len.append(length)
        self.seg_fresh.append(bool(fresh))

    def segments(self):
        return {"req": np.asarray(self.seg_req, np.int64), "kind": list(self.seg_kind),
                "key": list(self.seg_key), "start": np.asarray(self.seg_start, np.int64),
                "len": np.asarray(self.seg_len, np.int64),
                "fresh": np.asarray(self.seg_fresh, bool), "word_tables": self.word_tables}

    def build(self, R, device):
        seg_req = np.asarray(self.seg_req, np.int64)
        seg_len = np.asarray(self.seg_len, np.int64)
        lens = np.bincount(seg_req, weights=seg_len, minlength=R).astype(np.int64)
        tok_off = np.zeros(R + 1, np.int64)
        np.cumsum(lens, out=tok_off[1:])
        # segments are appended per request in order, so a stable sort by request keeps order
        order = np.argsort(seg_req, kind="stable")
        seg_len_o = seg_len[order]
        seg_pos = np.zeros(len(order) + 1, np.int64)
        np.cumsum(seg_len_o, out=seg_pos[1:])
        T = int(tok_off[-1])
        # word segments are gathered from one concatenated table
        tables = list(self.word_tables.items())
        tab_base = {}
        cat = []
        base = 0
        for k, arr in tables:
            tab_base[k] = base
            cat.append(arr)
            base += len(arr)
        word_tab = torch.from_numpy(np.concatenate(cat) if cat else np.zeros(1, np.int64)).to(device)
        kinds = [self.seg_kind[i] for i in order]
        keys = [self.seg_key[i] for i in order]
        starts = np.asarray([self.seg_start[i] for i in order], np.int64)
        is_word = np.array([k == "w" for k in kinds], bool)
        kh = np.array([0 if k == "w" else _signed(v) for k, v in zip(kinds, keys)], np.int64)
        wb = np.array([tab_base[v] if k == "w" else 0 for k, v in zip(kinds, keys)], np.int64)
        seg_of_tok = torch.repeat_interleave(torch.arange(len(order), device=device),
                                             torch.from_numpy(seg_len_o).to(device))
        pos_in_seg = torch.arange(T, device=device) - torch.from_numpy(seg_pos[:-1]).to(device)[seg_of_tok]
        idx = torch.from_numpy(starts).to(device)[seg_of_tok] + pos_in_seg
        toks = fnv1a_u64_vec(idx, torch.from_numpy(kh).to(device)[seg_of_tok])
        wmask = torch.from_numpy(is_word).to(device)[seg_of_tok]
        if bool(wmask.any()):
            widx = torch.from_numpy(wb).to(device)[seg_of_tok] + idx
            toks = torch.where(wmask, word_tab[torch.where(wmask, widx, 0)], toks)
        return toks, tok_off


def deep_research(n_workflows=10_000, seed=1, device=None, unprofiled_frac=0.1,
                  rounds=3, fanout=(2, 3), salt_tokens=4, task_tokens=256, wf_base=0,
                  model_stride=0) -> Trace:
    """Config 2 (BASELINE.json configs[1]): (decomposer -> researcher^{||2,3})^{3,3} ->
    summarizer -> critic -> writer -> verifier -> terminal; 6 roles on 2 models."""
    device = device or ("cuda" if torch.cuda.is_available() else "cpu")
    roles = [Role("decomposer", 0, 512, 0, 300, 0.3), Role("researcher", 0, 768, 1024, 1500, 0.45),
             Role("summarizer", 0, 512, 2048, 1200, 0.35), Role("critic", 1, 384, 1536, 600, 0.4),
             Role("writer", 1, 640, 2048, 2000, 0.4), Role("verifier", 1, 384, 1024, 300, 0.3)]
    rng = np.random.default_rng(seed)
    b = _Builder()
    res, group, wfs, rls = [], [], [], []
    r = 0
    for w in range(wf_base, wf_base + n_workflows):
        wid = f"w{w}"
        # model_stride > 0: workflow w runs on model pair 2*(w % model_stride) (+0/+1 by role)
        mbase = 2 * (w % model_stride) if model_stride else 0
        stages = []
        for _ in range(rounds):
            stages.append((0, 1))
            stages.append((1, int(rng.integers(fanout[0], fanout[1] + 1))))
        stages += [(2, 1), (3, 1), (4, 1), (5, 1)]
        prev_first, prev_out = None, 0
        for si, (ro, count) in enumerate(stages):
            role = roles[ro]
            outs = _lognormal(rng, role.out_mean, role.out_cv, count)
            first_rid = None
            for sib in range(count):
                rid = f"{wid}_s{si}_{sib}"
                if sib == 0:
                    first_rid = rid
                b.add(r, "w", b.words(f"sys_{role.name}", role.sys_tokens), 0, role.sys_tokens)
                if prev_first is not None:
                    b.add(r, "i", response_key(prev_first), 0, min(role.carry_tokens, prev_out))
                if si == 0:
                    b.add(r, "i", task_key(wid), 0, task_tokens, fresh=True)
                b.add(r, "i", salt_key(rid), 0, salt_tokens, fresh=True)
                plen = role.sys_tokens + (min(role.carry_tokens, prev_out) if prev_first else 0) + \
                    (task_tokens if si == 0 else 0) + salt_tokens
                if rng.random() < unprofiled_frac:
                    res.append((plen, GLOBAL_MAX_OUTPUT, 0.0, 0))
                else:
                    res.append((plen, _p99(role.out_mean, role.out_cv), ALPHA, 0))
                group.append(role.model + mbase)
                wfs.append(w)
                rls.append(ro)
                r += 1
            prev_first, prev_out = first_rid, int(outs[0])
    toks, tok_off = b.build(r, device)
    return _with_segments(b, Trace(toks, tok_off, np.array(res, RES_DTYPE), np.array(group, np.int32),
                 np.array(wfs, np.int32), np.array(rls, np.int32), roles,
                 2 * max(model_stride, 1), "deep_research"))


def coding_assistant(n_workflows=1_000, seed=1, device=None, unprofiled_frac=0.0) -> Trace:
    """Config 1: planner -> (explorer)^{||3,4} -> (engineer)^{3,6} -> reviewer -> terminal,
    Table-1 lengths; engineer re-sends its previous request + response
    (chat_accumulate, engine.cpp:362-374)."""
    device = device or ("cuda" if torch.cuda.is_available() else "cpu")
    roles = [Role("planner", 0, 300, 0, 60, 0.15), Role("explorer", 0, 600, 512, 1924, 0.45),
             Role("engineer", 0, 800, 1024, 3152, 0.45), Role("reviewer", 0, 500, 2048, 2620, 0.18)]
    rng = np.random.default_rng(seed)
    b = _Builder()
    res, group, wfs, rls = [], [], [], []
    r = 0
    for w in range(n_workflows):
        wid = f"w{w}"
        stages = [(0, 1), (1, int(rng.integers(3, 5)))] + [(2, 1)] * int(rng.integers(3, 7)) + [(3, 1)]
        prev_first, prev_out = None, 0
        last_eng = None  # (segments, response key, out_len)
        for si, (ro, count) in enumerate(stages):
            role = roles[ro]
            outs = _lognormal(rng, role.out_mean, role.out_cv, count)
            first_rid = None
            for sib in range(count):
                rid = f"{wid}_s{si}_{sib}"
                first_rid = first_rid or rid
                segs = []
                if ro == 2 and last_eng is not None:
                    segs = list(last_eng[0])
                    segs.append(("i", last_eng[1], 0, last_eng[2]))
                    segs.append(("w", b.words("turn_engineer", 8), 0, 8))
                else:
                    segs.append(("w", b.words(f"sys_{role.name}", role.sys_tokens), 0, role.sys_tokens))
                    if prev_first is not None:
                        segs.append(("i", response_key(prev_first), 0, min(role.carry_tokens, prev_out)))
                if si == 0:
                    segs.append(("i", task_key(wid), 0, 64))
                segs.append(("i", salt_key(rid), 0, 4))
                plen = 0
                for s in segs:
                    b.add(r, *s)
                    plen += s[3]
                if ro == 2:  # the next engineer turn re-sends this whole request + response
                    last_eng = (segs, response_key(rid), int(outs[sib]))
                if rng.random() < unprofiled_frac:
                    res.append((plen, GLOBAL_MAX_OUTPUT, 0.0, 0))
                else:
                    res.append((plen, _p99(role.out_mean, role.out_cv), ALPHA, 0))
                group.append(0)
                wfs.append(w)
                rls.append(ro)
                r += 1
            prev_first, prev_out = first_rid, int(outs[0])
    toks, tok_off = b.build(r, device)
    return _with_segments(b, Trace(toks, tok_off, np.array(res, RES_DTYPE), np.array(group, np.int32),
                 np.array(wfs, np.int32), np.array(rls, np.int32), roles, 1, "coding_assistant"))


def long_context(n_requests=100_000, seed=1, device=None, n_roles=8, steps=4,
                 sys_tokens=2048, ctx_tokens=28672, unique_tokens=2048, r_base=0,
                 n_keep=None) -> Trace:
    """Config 3: L = 32,768 = 2,048-token role sys prompt + 28,672-token per-workflow carried
    context (shared by the workflow's `steps` requests) + 2,048 unique tokens.  r_base offsets
    request / workflow ids (a later burst of the trace); n_keep keeps the first n_keep."""
    device = device or ("cuda" if torch.cuda.is_available() else "cpu")
    rng = np.random.default_rng(seed)
    b = _Builder()
    roles = [Role(f"role{k}", 0, sys_tokens, ctx_tokens, 1000, 0.45) for k in range(n_roles)]
    res, group, wfs, rls = [], [], [], []
    up = _p99(1000, 0.45)
    if n_keep is not None:
        n_requests = min(n_requests, n_keep)
    for r in range(n_requests):
        g = r_base + r
        w = g // steps
        ro = int(rng.integers(0, n_roles))
        b.add(r, "w", b.words(f"sys_role{ro}", sys_tokens), 0, sys_tokens)
        b.add(r, "i", response_key(f"w{w}_ctx"), 0, ctx_tokens)
        b.add(r, "i", salt_key(f"w{w}_s{g % steps}_0"), 0, unique_tokens, fresh=True)
        res.append((sys_tokens + ctx_tokens + unique_tokens, up, ALPHA, 0))
        group.append(0)
        wfs.append(w)
        rls.append(ro)
    toks, tok_off = b.build(n_requests, device)
    return _with_segments(b, Trace(toks, tok_off, np.array(res, RES_DTYPE), np.array(group, np.int32),
                 np.array(wfs, np.int32), np.array(rls, np.int32), roles, 1, "long_context"))


def bursty(n_requests=1_000_000, seed=1, device=None, n_models=4, mean_len=2048, cv=1.0,
           n_prefixes=512, r_base=0, n_keep=None) -> Trace:
    """Config 4: L ~ lognormal(2048, 1.0) clamped to [64, 32768] over 4 models; prompts share
    one of n_prefixes system prefixes (shared across the model's workflows) + unique suffix.
    r_base offsets request / workflow ids (one GPU's slice of a larger burst).  n_keep: only
    the first n_keep requests of the n_requests drawn (a bounded sample whose requests equal
    the full burst's first n_keep)."""
    device = device or ("cuda" if torch.cuda.is_available() else "cpu")
    rng = np.random.default_rng(seed)
    s2 = math.log(1 + cv * cv)
    L = np.clip(np.rint(rng.lognormal(math.log(mean_len) - s2 / 2, math.sqrt(s2), n_requests)), 64,
                32768).astype(np.int64)
    model = rng.integers(0, n_models, n_requests).astype(np.int32)
    pre = rng.integers(0, n_prefixes, n_requests)
    plen = np.minimum(L // 2, 1024 + (pre % 4) * 256)
    b = _Builder()
    pkeys = [fnv1a_str(f"prefix{p}") for p in range(n_prefixes)]
    up = _p99(500, 0.5)
    unprof = rng.random(n_requests) < 0.1
    if n_keep is not None and n_keep < n_requests:
        n_requests = n_keep
        L, model, pre, plen, unprof = L[:n_keep], model[:n_keep], pre[:n_keep], plen[:n_keep], \
            unprof[:n_keep]
    for r in range(n_requests):
        b.add(r, "i", pkeys[pre[r]], 0, int(plen[r]))
        b.add(r, "i", salt_key(f"b{r_base + r}"), 0, int(L[r] - plen[r]), fresh=True)
    res = np.zeros(n_requests, RES_DTYPE)
    res["prompt_len"] = L
    res["upper"] = np.where(unprof, GLOBAL_MAX_OUTPUT, up)
    res["alpha"] = np.where(unprof, 0.0, ALPHA)
    toks, tok_off = b.build(n_requests, device)
    return _with_segments(b, Trace(toks, tok_off, res, model,
                 ((r_base + np.arange(n_requests)) // 8).astype(np.int32),
                 (pre % 16).astype(np.int32), [], n_models, "bursty"))


@dataclass
class Cluster:
    """Replica layout + background load of one GPU's shard (NodeView inputs)."""
    n_replicas: int
    model_of: np.ndarray          # int32 [n]
    replica_id: np.ndarray        # int32 [n]
    kv_capacity: np.ndarray       # int64 [n]
    l2_capacity: np.ndarray       # int64 [n]
    asg_off: np.ndarray           # int64 [n+1]
    asg: np.ndarray               # RES_DTYPE
    cand_off: np.ndarray          # int32 [G+1]  candidates per model, ascending replica id
    cand: np.ndarray              # int32


def make_cluster(n_replicas, n_models, kv=100_000, l2=200_000, seed=0, max_bg=3, id_base=0,
                 interleave=False):
    """n_replicas replicas of n_models models: contiguous blocks of replicas per model, or
    (interleave) replica i serves model i % n_models."""
    rng = np.random.default_rng(seed)
    if interleave:
        model_of = (np.arange(n_replicas) % max(n_models, 1)).astype(np.int32)
    else:
        model_of = (np.arange(n_replicas) * n_models // max(n_replicas, 1)).astype(np.int32)
    asg, off = [], [0]
    for n in range(n_replicas):
        k = int(rng.integers(0, max_bg + 1))
        for _ in range(k):
            asg.append((int(rng.integers(500, 3000)), int(rng.integers(500, 3000)), ALPHA, 0))
        off.append(len(asg))
    cand = np.concatenate([np.nonzero(model_of == m)[0] for m in range(n_models)]).astype(np.int32)
    cand_off = np.zeros(n_models + 1, np.int32)
    np.cumsum(np.bincount(model_of, minlength=n_models), out=cand_off[1:])
    return Cluster(n_replicas, model_of, (np.arange(n_replicas) + id_base).astype(np.int32),
                   np.full(n_replicas, kv, np.int64), np.full(n_replicas, l2, np.int64),
                   np.array(off, np.int64), np.array(asg, RES_DTYPE) if asg else np.zeros(0, RES_DTYPE),
                   cand_off, cand)
