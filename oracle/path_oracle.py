"""TEST INFRASTRUCTURE ONLY (parity checker for K6, csrc/k_nextuse.cu).

Pure-Python restatement of the reference's next-use analysis over a FLATTENED path
expression (preorder node table, the layout of pyg_path_node in include/pyg.h):

  remaining_expr(cursor)           path_analysis.cpp:257-290
  first_occurrence(node, role)     path_analysis.cpp:408-444  (seq_compose :374-386, mix :388-404)
  repeat/fanout continue probs     path_analysis.cpp:14-24
  expected_distance_to             path_analysis.cpp:553-557
  future_roles / collect_reachable path_analysis.cpp:338-360, 547-551

Python floats are IEEE doubles evaluated in source order, as the reference's x86-64
build (no FMA contraction) evaluates them, so values are bit-identical; pinned by
tests/golden/nextuse_golden.json (made by tests/golden/make_nextuse_golden.py with the
reference itself) in tests/test_nextuse.py.
"""
from __future__ import annotations

ATOM, SEQ, REPEAT, FANOUT, OPTIONAL, TERMINAL = range(6)  # path_expr.hpp PathKind order


class Node:
    __slots__ = ("kind", "role", "min", "max", "p_continue", "p", "child", "children")

    def __init__(self, kind, role=-1, mn=0, mx=0, p_continue=0.5, p=0.5, child=-1, children=()):
        self.kind, self.role, self.min, self.max = kind, role, mn, mx
        self.p_continue, self.p, self.child, self.children = p_continue, p, child, list(children)


def _fo_default():
    return [1.0, 0.0, 0.0, 0.0]  # FirstOcc{}: p_none, e_len_none, p_some, e_first


def seq_compose(a, b):
    r = _fo_default()
    r[2] = a[2] + a[0] * b[2]
    if r[2] > 0.0:
        r[3] = (a[2] * a[3] + a[0] * b[2] * (a[1] + b[3])) / r[2]
    r[0] = a[0] * b[0]
    r[1] = a[1] + b[1] if r[0] > 0.0 else 0.0
    return r


def mix(branches):
    r = _fo_default()
    r[0] = 0.0
    first_acc = none_len_acc = 0.0
    for w, occ in branches:
        r[2] += w * occ[2]
        first_acc += w * occ[2] * occ[3]
        r[0] += w * occ[0]
        none_len_acc += w * occ[0] * occ[1]
    if r[2] > 0.0:
        r[3] = first_acc / r[2]
    if r[0] > 0.0:
        r[1] = none_len_acc / r[0]
    return r


def repeat_continue_prob(m, mx, q, done):
    if done < m:
        return 1.0
    if done >= mx:
        return 0.0
    return q


def fanout_continue_prob(a, b, done):
    if done < a:
        return 1.0
    if done >= b:
        return 0.0
    return float(b - done) / float(b - done + 1)


def loop_occ(is_repeat, mn, mx, q, child):
    branches = []
    prefix = _fo_default()
    reach = 1.0
    for done in range(0, mx + 1):
        cont = repeat_continue_prob(mn, mx, q, done) if is_repeat else fanout_continue_prob(mn, mx, done)
        stop = reach * (1.0 - cont)
        if stop > 0.0:
            branches.append((stop, prefix))
        reach *= cont
        if reach <= 0.0:
            break
        prefix = seq_compose(prefix, child)
    return mix(branches)


def first_occurrence(nodes, i, role):
    n = nodes[i]
    if n.kind == TERMINAL:
        return _fo_default()
    if n.kind == ATOM:
        return [0.0, 0.0, 1.0, 1.0] if n.role == role else [1.0, 1.0, 0.0, 0.0]
    if n.kind == SEQ:
        acc = _fo_default()
        for c in n.children:
            acc = seq_compose(acc, first_occurrence(nodes, c, role))
        return acc
    if n.kind == OPTIONAL:
        return mix([(1.0 - n.p, _fo_default()), (n.p, first_occurrence(nodes, n.child, role))])
    return loop_occ(n.kind == REPEAT, n.min, n.max, n.p_continue,
                    first_occurrence(nodes, n.child, role))


def reachable(nodes, i):
    """collect_reachable as a role bitmask."""
    n = nodes[i]
    if n.kind == TERMINAL:
        return 0
    if n.kind == ATOM:
        return 1 << n.role
    if n.kind == SEQ:
        m = 0
        for c in n.children:
            m |= reachable(nodes, c)
        return m
    if n.kind == OPTIONAL:
        return reachable(nodes, n.child) if n.p > 0.0 else 0
    if n.kind == REPEAT:
        ok = n.max >= 1 and (n.min >= 1 or n.p_continue > 0.0)
        return reachable(nodes, n.child) if ok else 0
    return reachable(nodes, n.child) if n.max >= 1 else 0  # FANOUT


def remaining_pieces(nodes, frames):
    """remaining_expr: ('node', i) or ('repeat', child, rem_min, rem_max, q), in order."""
    pieces = []
    for idx in range(len(frames) - 2, -1, -1):
        node_i, prog = frames[idx]
        n = nodes[node_i]
        if n.kind == SEQ:
            for c in n.children[prog + 1:]:
                pieces.append(("node", c))
        elif n.kind == REPEAT:
            done = prog + 1
            rem_max = n.max - done
            if rem_max > 0:
                pieces.append(("repeat", n.child, max(n.min - done, 0), rem_max, n.p_continue))
    return pieces


def expected_distance_to(nodes, frames, role):
    acc = _fo_default()
    for pc in remaining_pieces(nodes, frames):
        if pc[0] == "node":
            occ = first_occurrence(nodes, pc[1], role)
        else:
            occ = loop_occ(True, pc[2], pc[3], pc[4], first_occurrence(nodes, pc[1], role))
        acc = seq_compose(acc, occ)
    return acc[3] if acc[2] > 0.0 else None


def future_mask(nodes, frames):
    m = 0
    for pc in remaining_pieces(nodes, frames):
        if pc[0] == "node":
            m |= reachable(nodes, pc[1])
        else:
            _, child, rmin, rmax, q = pc
            if rmax >= 1 and (rmin >= 1 or q > 0.0):
                m |= reachable(nodes, child)
    return m


def from_table(table):
    """Node list from the flattened arrays (dict of lists, pyg_path_node fields)."""
    out = []
    ch = table["ch_list"]
    for i in range(len(table["kind"])):
        out.append(Node(table["kind"][i], table["role"][i], table["min"][i], table["max"][i],
                        table["p_continue"][i], table["p"][i], table["child"][i],
                        ch[table["ch_begin"][i]:table["ch_end"][i]]))
    return out
