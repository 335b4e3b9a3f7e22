"""Generates tests/golden/nextuse_golden.json from the REFERENCE itself (run here, where
/root/reference and oracle/_ref/libpythia_ref64.so exist):

  random flattened path expressions (+ the config-1/config-2 workflow shapes), random
  histories = prefixes of sampled words of each language, and for every located history
  the reference's cursor frames (locate_position), expected_distance_to for every role and
  future_roles (path_analysis.cpp), through the extern "C" shim in oracle/ref_shim.cpp.

    python tests/golden/make_nextuse_golden.py
"""
import ctypes as C
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.path_oracle import ATOM, FANOUT, OPTIONAL, REPEAT, SEQ, TERMINAL  # noqa: E402

N_ROLES = 6


class PNode(C.Structure):
    _fields_ = [("kind", C.c_int32), ("role", C.c_int32), ("min", C.c_int32), ("max", C.c_int32),
                ("p_continue", C.c_double), ("p", C.c_double), ("child", C.c_int32),
                ("ch_begin", C.c_int32), ("ch_end", C.c_int32), ("pad", C.c_int32)]


class Tree:
    def __init__(self):
        self.nodes = []   # dicts, preorder
        self.ch = []

    def add(self, **kw):
        d = dict(kind=TERMINAL, role=-1, min=0, max=0, p_continue=0.5, p=0.5, child=-1,
                 ch_begin=0, ch_end=0)
        d.update(kw)
        self.nodes.append(d)
        return len(self.nodes) - 1

    def table(self):
        keys = ["kind", "role", "min", "max", "p_continue", "p", "child", "ch_begin", "ch_end"]
        t = {k: [n[k] for n in self.nodes] for k in keys}
        t["ch_list"] = list(self.ch)
        return t


PROBS = [0.0, 0.25, 0.5, 0.7, 1.0]


def gen(rng, t, depth, allow_seq=True):
    """Preorder emission of a random non-terminal node."""
    r = rng.random()
    if depth <= 0 or r < 0.35:
        return t.add(kind=ATOM, role=rng.randrange(N_ROLES))
    if allow_seq and r < 0.55:
        i = t.add(kind=SEQ)
        kids = []
        for _ in range(rng.randint(2, 3)):
            kids.append(None)
        # children are emitted after the parent (preorder); the list is filled afterwards
        ids = [gen(rng, t, depth - 1, allow_seq=False) for _ in kids]
        t.nodes[i]["ch_begin"] = len(t.ch)
        t.ch.extend(ids)
        t.nodes[i]["ch_end"] = len(t.ch)
        return i
    kind = rng.choice([REPEAT, FANOUT, OPTIONAL])
    i = t.add(kind=kind)
    if kind == OPTIONAL:
        t.nodes[i]["p"] = rng.choice(PROBS)
    else:
        mn = rng.randint(0, 2)
        t.nodes[i]["min"] = mn
        t.nodes[i]["max"] = mn + rng.randint(0, 2)
        if kind == REPEAT:
            t.nodes[i]["p_continue"] = rng.choice(PROBS)
    t.nodes[i]["child"] = gen(rng, t, depth - 1, allow_seq=True)
    return i


def random_expr(rng):
    t = Tree()
    root = t.add(kind=SEQ)
    ids = [gen(rng, t, 3, allow_seq=False) for _ in range(rng.randint(1, 4))]
    ids.append(t.add(kind=TERMINAL))
    # the root's children must be contiguous in ch_list: ch is only appended by nested seqs,
    # which were emitted while generating `ids`, so append the root's list now
    t.nodes[root]["ch_begin"] = len(t.ch)
    t.ch.extend(ids)
    t.nodes[root]["ch_end"] = len(t.ch)
    return t


def workflow_expr(kind):
    """config-2: (decomposer -> (researcher)^{||2,3})^{3,3} -> summarizer -> critic -> writer
    -> verifier -> terminal; config-1: planner -> (explorer)^{||3,4} -> (engineer)^{3,6} ->
    reviewer -> terminal (roles numbered in order)."""
    t = Tree()
    root = t.add(kind=SEQ)
    ids = []
    if kind == "deep_research":
        rep = t.add(kind=REPEAT, min=3, max=3, p_continue=0.5)
        seq = t.add(kind=SEQ)
        a = t.add(kind=ATOM, role=0)
        f = t.add(kind=FANOUT, min=2, max=3)
        b = t.add(kind=ATOM, role=1)
        t.nodes[f]["child"] = b
        t.nodes[seq]["ch_begin"] = len(t.ch)
        t.ch.extend([a, f])
        t.nodes[seq]["ch_end"] = len(t.ch)
        t.nodes[rep]["child"] = seq
        ids = [rep] + [t.add(kind=ATOM, role=k) for k in (2, 3, 4, 5)]
    else:
        ids.append(t.add(kind=ATOM, role=0))
        f = t.add(kind=FANOUT, min=3, max=4)
        t.nodes[f]["child"] = t.add(kind=ATOM, role=1)
        ids.append(f)
        r = t.add(kind=REPEAT, min=3, max=6, p_continue=0.5)
        t.nodes[r]["child"] = t.add(kind=ATOM, role=2)
        ids.append(r)
        ids.append(t.add(kind=ATOM, role=3))
    ids.append(t.add(kind=TERMINAL))
    t.nodes[root]["ch_begin"] = len(t.ch)
    t.ch.extend(ids)
    t.nodes[root]["ch_end"] = len(t.ch)
    return t


def sample_word(rng, t, i):
    n = t.nodes[i]
    k = n["kind"]
    if k == TERMINAL:
        return []
    if k == ATOM:
        return [n["role"]]
    if k == SEQ:
        out = []
        for c in t.ch[n["ch_begin"]:n["ch_end"]]:
            out += sample_word(rng, t, c)
        return out
    if k == OPTIONAL:
        return sample_word(rng, t, n["child"]) if rng.random() < n["p"] else []
    if k == REPEAT:
        cnt = n["min"]
        while cnt < n["max"] and rng.random() < n["p_continue"]:
            cnt += 1
    else:
        cnt = rng.randint(n["min"], n["max"])
    out = []
    for _ in range(cnt):
        out += sample_word(rng, t, n["child"])
    return out


def main():
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libpythia_ref64.so"))
    lib.pref_path_build.restype = C.c_void_p
    lib.pref_path_build.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
    lib.pref_path_free.argtypes = [C.c_void_p]
    lib.pref_path_locate.restype = C.c_int32
    lib.pref_path_locate.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                     C.c_int32]
    lib.pref_path_distance.restype = C.c_int32
    lib.pref_path_distance.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                       C.c_void_p]
    rng = random.Random(2604)
    cases = []
    trees = [workflow_expr("deep_research"), workflow_expr("coding")] + \
        [random_expr(rng) for _ in range(160)]
    for t in trees:
        tab = t.table()
        n = len(t.nodes)
        arr = (PNode * n)(*[PNode(d["kind"], d["role"], d["min"], d["max"], d["p_continue"],
                                  d["p"], d["child"], d["ch_begin"], d["ch_end"], 0)
                            for d in t.nodes])
        ch = (C.c_int32 * max(len(t.ch), 1))(*t.ch)
        h = lib.pref_path_build(arr, ch, 0)
        if not h:
            continue
        queries = []
        seen = set()
        for _ in range(12):
            w = sample_word(rng, t, 0)
            for L in range(1, len(w) + 1):
                hist = tuple(w[:L])
                if hist in seen:
                    continue
                seen.add(hist)
                hh = (C.c_int32 * L)(*hist)
                fn = (C.c_int32 * 64)()
                fp = (C.c_int32 * 64)()
                nf = lib.pref_path_locate(h, hh, L, fn, fp, 64)
                if nf < 0:
                    continue
                dist = []
                mask = C.c_uint64()
                for role in range(N_ROLES):
                    d = C.c_double()
                    rc = lib.pref_path_distance(h, hh, L, role, C.byref(d), C.byref(mask))
                    dist.append(d.value.hex() if rc == 0 else None)
                queries.append({"history": list(hist),
                                "frames": [[fn[k], fp[k]] for k in range(nf)],
                                "distance": dist, "future_mask": mask.value})
        lib.pref_path_free(h)
        if queries:
            cases.append({"table": tab, "queries": queries})
    out = os.path.join(ROOT, "tests", "golden", "nextuse_golden.json.gz")
    import gzip
    with gzip.open(out, "wt") as f:
        json.dump({"source": "reference path_analysis.cpp via oracle/ref_shim.cpp",
                   "n_roles": N_ROLES, "cases": cases}, f, separators=(",", ":"))
    nq = sum(len(c["queries"]) for c in cases)
    print(f"wrote {out}: {len(cases)} expressions, {nq} located histories")


if __name__ == "__main__":
    main()
