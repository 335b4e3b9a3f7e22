"""Prompt templates on the device: the host side of pyg_assemble_dev.

A reference prompt template (prompt.hpp:17-36) interleaves literal words with exact
references into earlier exchanges, in the text form "${req_12:request:[0,250]}".  Serving
keeps every exchange in HBM, so assembling a prompt is a gather: the host resolves each
template to (pool offset, length) segments -- clamping references to what exists,
tokenizing literal words -- and ships only those descriptors plus the literal tokens;
pyg_assemble_dev builds the token CSR on the device.

  parse(text)            parse_prompt_template (prompt.cpp:75-101), same errors (ValueError)
  tokenize_words(text)   prompt.cpp:11-21: C-locale whitespace split, fnv1a(word)
  ExchangePool           exchanges (request, response tokens) resident in a device pool
  ExchangePool.resolve   assemble_prompt (prompt.cpp:128-142) / assemble_resolvable_prefix
                         (:144-164) semantics as segments
  ExchangePool.assemble  a batch of templates -> token CSR on the device
"""
from __future__ import annotations

import ctypes as C
import re
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check
from .workload import FNV_OFFSET, FNV_PRIME, M64

_WS = re.compile(rb"[ \t\n\v\f\r]+")  # std::isspace in the C locale


def _fnv_bytes(b: bytes) -> int:
    """fnv1a(std::string_view) (tokens.hpp:22-28) over the word's bytes."""
    h = FNV_OFFSET
    for c in b:
        h = ((h ^ c) * FNV_PRIME) & M64
    return h


def tokenize_words(text: str) -> np.ndarray:
    words = [w for w in _WS.split(text.encode()) if w]
    return np.array([_fnv_bytes(w) for w in words], np.uint64)


@dataclass
class Ref:
    request_id: str
    response: bool
    start: int
    end: int


def _stoll(s: str) -> int:
    """std::stoll: leading whitespace, optional sign, digits (at least one); the rest ignored."""
    m = re.match(r"[ \t\n\v\f\r]*([+-]?[0-9]+)", s)
    if not m:
        raise ValueError("stoll: no conversion")
    v = int(m.group(1))
    if not -(1 << 63) <= v < (1 << 63):
        raise ValueError("stoll: out of range")
    return v


def _placeholder(body: str) -> Ref:
    c1 = body.find(":")
    c2 = body.find(":", c1 + 1) if c1 >= 0 else -1
    if c1 < 0 or c2 < 0:
        raise ValueError("malformed placeholder: " + body)
    source = body[c1 + 1:c2]
    if source not in ("request", "response"):
        raise ValueError("placeholder source must be request|response: " + body)
    rng = body[c2 + 1:]
    if len(rng) < 5 or rng[0] != "[" or rng[-1] != "]":
        raise ValueError("malformed placeholder range: " + body)
    comma = rng.find(",")
    if comma < 0:
        raise ValueError("malformed range: " + body)
    start = _stoll(rng[1:comma])
    end = _stoll(rng[comma + 1:len(rng) - 1])
    if start < 0 or start >= end:
        raise ValueError("range must satisfy 0 <= start < end: " + body)
    return Ref(body[:c1], source == "response", start, end)


def parse(text: str) -> list:
    """Segments: str (a literal run) or Ref, in order."""
    segs, lit, i = [], [], 0
    while i < len(text):
        if text[i] == "$" and i + 1 < len(text) and text[i + 1] == "{":
            close = text.find("}", i + 2)
            if close < 0:
                raise ValueError("unterminated placeholder")
            if lit:
                segs.append("".join(lit))
                lit = []
            segs.append(_placeholder(text[i + 2:close]))
            i = close + 1
        else:
            lit.append(text[i])
            i += 1
    if lit:
        segs.append("".join(lit))
    return segs


class ExchangePool:
    """Exchanges resident in one device token pool: id -> (request, response) ranges."""

    def __init__(self, exchanges: dict, device="cuda"):
        self.where = {}
        parts, off = [], 0
        for rid, (req, resp) in exchanges.items():
            req = np.asarray(req, np.uint64)
            resp = np.asarray(resp, np.uint64)
            self.where[rid] = (off, len(req), off + len(req), len(resp))
            parts += [req, resp]
            off += len(req) + len(resp)
        flat = np.concatenate(parts) if parts else np.zeros(0, np.uint64)
        self.n_resident = off
        self.host = flat
        self.device = device
        self.pool = torch.from_numpy(flat.view(np.int64).copy()).to(device) if off else \
            torch.zeros(1, dtype=torch.int64, device=device)

    def resolve(self, tmpl, prefix=False):
        """[(kind, a, b)] with kind 'p' (pool offset a, length b) or 'l' (literal tokens a),
        and complete.  None when assemble_prompt would return nullopt."""
        segs = parse(tmpl) if isinstance(tmpl, str) else tmpl
        out = []
        for s in segs:
            if isinstance(s, str):
                toks = tokenize_words(s)
                if len(toks):
                    out.append(("l", toks, len(toks)))
                continue
            w = self.where.get(s.request_id)
            if w is None:
                if prefix:
                    return out, False
                return None
            base, n = (w[2], w[3]) if s.response else (w[0], w[1])
            lo, hi = min(s.start, n), min(s.end, n)  # append_slice clamps (prompt.cpp:117-123)
            if hi > lo:
                out.append(("p", base + lo, hi - lo))
        return out, True

    def gather_host(self, resolved) -> np.ndarray:
        parts = [a if k == "l" else self.host[a:a + b] for k, a, b in resolved]
        return np.concatenate(parts) if parts else np.zeros(0, np.uint64)

    def assemble(self, ctx, resolved_list):
        """Token CSR (tok_off int64 [R+1], tokens) on the device for a batch of resolved
        templates: literal tokens go to a fresh region after the resident pool, every
        segment becomes a (pool offset, length) descriptor, pyg_assemble_dev gathers."""
        R = len(resolved_list)
        lits = [a for res in resolved_list for k, a, _ in res if k == "l"]
        lit_flat = np.concatenate(lits) if lits else np.zeros(0, np.uint64)
        pool = torch.cat([self.pool[:max(self.n_resident, 0)],
                          torch.from_numpy(lit_flat.view(np.int64).copy()).to(self.device),
                          torch.zeros(1, dtype=torch.int64, device=self.device)])
        segs, seg_off, lpos = [], [0], self.n_resident
        for res in resolved_list:
            for k, a, b in res:
                if k == "l":
                    segs.append((lpos, b))
                    lpos += b
                else:
                    segs.append((a, b))
            seg_off.append(len(segs))
        d_segs = torch.tensor(segs if segs else [(0, 0)], dtype=torch.int64, device=self.device)
        d_seg_off = torch.tensor(seg_off, dtype=torch.int64, device=self.device)
        n_tok = int(sum(b for s in segs for b in [s[1]]))
        tok_off = torch.zeros(R + 1, dtype=torch.int64, device=self.device)
        tokens = torch.zeros(max(n_tok, 1), dtype=torch.int64, device=self.device)
        check(_lib._lib.pyg_assemble_dev(ctx.h, R, C.c_void_p(d_seg_off.data_ptr()),
                                         C.c_void_p(d_segs.data_ptr()),
                                         C.c_void_p(pool.data_ptr()),
                                         C.c_void_p(tok_off.data_ptr()),
                                         C.c_void_p(tokens.data_ptr())))
        return tok_off, tokens


__all__ = ["parse", "tokenize_words", "Ref", "ExchangePool"]
