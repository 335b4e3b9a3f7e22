"""K6 oracle (oracle/path_oracle.py) pinned against the reference's own next-use values
(tests/golden/nextuse_golden.json.gz, made by make_nextuse_golden.py through the compiled
reference), bit for bit; and against the live reference when oracle/_ref is built."""
import gzip
import json
import os

import pytest

from oracle import path_oracle as P

GOLD = os.path.join(os.path.dirname(__file__), "golden", "nextuse_golden.json.gz")


def _gold():
    with gzip.open(GOLD, "rt") as f:
        return json.load(f)


def test_golden_is_substantial():
    g = _gold()
    nq = sum(len(c["queries"]) for c in g["cases"])
    defined = sum(d is not None for c in g["cases"] for q in c["queries"] for d in q["distance"])
    assert len(g["cases"]) >= 100 and nq >= 1000 and defined >= 1000


def test_restatement_matches_reference_golden_bit_exact():
    g = _gold()
    for ci, c in enumerate(g["cases"]):
        nodes = P.from_table(c["table"])
        for q in c["queries"]:
            fr = [tuple(x) for x in q["frames"]]
            assert P.future_mask(nodes, fr) == q["future_mask"], (ci, q["history"])
            for role in range(g["n_roles"]):
                d = P.expected_distance_to(nodes, fr, role)
                w = q["distance"][role]
                assert (d is None) == (w is None), (ci, q["history"], role)
                if d is not None:
                    assert d.hex() == w, (ci, q["history"], role, d, float.fromhex(w))


def test_liveness_equals_defined_next_use():
    """future_roles(c) contains r  <=>  expected_distance_to(c, r) is defined."""
    g = _gold()
    for c in g["cases"]:
        for q in c["queries"]:
            for role in range(g["n_roles"]):
                assert ((q["future_mask"] >> role) & 1) == (q["distance"][role] is not None)
