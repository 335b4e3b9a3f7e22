"""Pins the C restatement oracle (oracle/pyg_oracle.c) before anything is
checked against it:

1. the reference's own known-answer tests, replayed case by case
   (tests/test_cache.cpp, tests/test_sched.cpp under /root/reference/proj),
   including the seeded random trials via a bit-exact std::mt19937_64;
2. hash KATs measured on the reference;
3. randomized differential runs against the reference's own implementation
   (oracle/_ref, compiled unmodified) when that library is present.

CPU only.
"""
import numpy as np
import pytest

from mt64 import MT19937_64
from oracle.py_oracle import Reference, Restated, reference_available

L1, L2, L3 = 0, 1, 2


def make_tokens(salt, n):
    # tests/test_cache.cpp:19-23
    return np.array([(salt * 1_000_003 + i) & ((1 << 64) - 1) for i in range(n)], np.uint64)


BACKENDS = [("restated", lambda B: Restated(B))]
if reference_available(64):
    BACKENDS.append(("reference", lambda B: Reference(B)))


@pytest.fixture(params=[b[0] for b in BACKENDS])
def be64(request):
    return dict(BACKENDS)[request.param](64)


# ---------------------------------------------------------------- hashing KATs
def test_fnv_kats(restated64):
    o = restated64
    assert o.fnv1a_str("") == 0x14650FB0739D0383  # non-standard offset (tokens.hpp:19)
    assert o.fnv1a_str("a") == 0x44BD8AD473CD9906
    assert o.fnv1a_str("a") != 0xAF63DC4C8601EC8C  # standard FNV-1a vector must NOT hold
    assert o.fnv1a_u64(0) == 0x47FE0D7EAF8E51E3
    assert o.fnv1a_u64(1) == 0x29034675A49F07C2


def test_chain_hash_kat_b64_b16():
    t = np.arange(150, dtype=np.uint64)
    h64 = Restated(64).chain_hashes(t)
    assert [int(x) for x in h64] == [0x9C4E47906FA54D83, 0x3A93E08760069B83, 0x70F20F295E45E2A2]
    h16 = Restated(16).chain_hashes(t)
    assert len(h16) == 10
    assert h16[3] == h64[0] and h16[7] == h64[1] and h16[9] == h64[2]


def test_chain_hash_edge_cases(restated16):
    o = restated16
    assert len(o.chain_hashes(np.zeros(0, np.uint64))) == 0
    assert len(o.chain_hashes(np.zeros(1, np.uint64))) == 1
    assert len(o.chain_hashes(np.zeros(16, np.uint64))) == 1
    assert len(o.chain_hashes(np.zeros(17, np.uint64))) == 2
    big = np.array([(1 << 64) - 1, 0x0123456789ABCDEF], np.uint64)
    h = o.fnv1a_u64(0x0123456789ABCDEF, o.fnv1a_u64((1 << 64) - 1))
    assert o.chain_hashes(big)[-1] == h


# ----------------------------------------------------- test_cache.cpp lookups
def test_lookup_empty(be64):
    c, l3 = be64.new_cache(10000, 10000), be64.new_l3()
    assert be64.lookup(c, l3, make_tokens(1, 300)) == (0, 0, 0)  # :41-48


def test_lookup_staged_l2(be64):
    c = be64.new_cache(10000, 10000)
    p = make_tokens(2, 500)
    be64.insert_chain(c, L2, p, 500, 0, 0, 1.0, 0)  # :50-58
    assert be64.lookup(c, None, p) == (0, 500, 0)
    assert be64.occupancy(c, None, L2) == 500


def test_lookup_ragged_and_divergence(be64):
    c = be64.new_cache(10000, 10000)  # :60-71
    be64.insert_chain(c, L1, make_tokens(3, 250), 250, 0, 0, 1.0, 0)
    assert be64.lookup(c, None, make_tokens(3, 600))[0] == 250
    d = make_tokens(3, 600)
    d[200] ^= np.uint64(0xFF)
    assert be64.lookup(c, None, d)[0] == 192


# -------------------------------------------------- test_cache.cpp completion
def test_completion_frees_dead_retains_live(be64):
    # :86-122 with roles planner=0 explorer=1 engineer=2 reviewer=3 verifier=4; wf w=0 other=1
    o = be64
    c, l3 = o.new_cache(100000, 100000), o.new_l3()
    pb, eb, ob = make_tokens(10, 128), make_tokens(11, 128), make_tokens(12, 64)
    o.insert_chain(c, L1, pb, 128, 0, 0, 1.0, 0)
    o.insert_chain(c, L1, eb, 128, 0, 1, 1.0, 0)
    o.insert_chain(c, L1, ob, 64, 1, 0, 1.0, 0)
    future = (1 << 1) | (1 << 2) | (1 << 3) | (1 << 4)  # future_nodes after planner
    if isinstance(o, Reference):
        expr = ("r0 -> (r1)^{||3,4} -> (r2)^{3,6} -> r3 -> (r2^{2-4} -> r3)? -> r4 -> terminal")
        assert o.future_mask(expr, ["r0"]) == future
    n = o.complete(c, l3, 0, future, 2.0)
    assert n == 4  # 2 frees + 2 retains
    assert o.lookup(c, l3, pb)[0] == 0
    assert o.lookup(c, l3, eb)[0] == 128
    assert o.lookup(c, l3, eb)[2] == 128
    assert o.lookup(c, l3, ob)[0] == 64


def test_completion_terminal_frees_all_unpinned(be64):
    o = be64  # :124-142, roles a=0 verifier=1
    c, l3 = o.new_cache(100000, 100000), o.new_l3()
    for i in range(5):
        o.insert_chain(c, L1 if i % 2 else L2, make_tokens(20 + i, 64), 64, 0, 0 if i % 2 else 1,
                       1.0, 0)
    pinned = make_tokens(40, 64)
    o.insert_chain(c, L1, pinned, 64, 0, 0, 1.0, 1)
    o.complete(c, l3, 0, 0, 2.0)
    assert o.occupancy(c, None, L1) == 64
    assert o.occupancy(c, None, L2) == 0
    assert o.lookup(c, l3, pinned)[0] == 64


def test_completion_unprofiled_noop(restated64):
    o = restated64
    c, l3 = o.new_cache(10000, 10000), o.new_l3()
    o.insert_chain(c, L1, make_tokens(5, 64), 64, 0, 0, 1.0, 0)
    assert o.complete(c, l3, 0, 0, 1.0, profiled=False) == 0


def test_completion_set_filter_oracle_seed71(be64):
    # :144-184 -- replays the reference's mt19937_64(71) trial states
    o = be64
    rng = MT19937_64(71)
    future = (1 << 1) | (1 << 2) | (1 << 3)  # future_roles after "a" in a -> b? -> (c)^{1,3} -> d
    if isinstance(o, Reference):
        assert o.future_mask("r0 -> r1? -> (r2)^{1,3} -> r3 -> terminal", ["r0"]) == future
    for trial in range(100):
        c, l3 = o.new_cache(1_000_000, 1_000_000), o.new_l3()
        placed = []
        for i in range(20):
            tier = L1 if rng() % 2 else L2
            wf = 0 if rng() % 2 else 1
            role = rng() % 5  # roles a,b,c,d,zz -> 0..4
            pin = tier == L1 and rng() % 4 == 0
            toks = make_tokens(1000 + trial * 100 + i, 64)
            o.insert_chain(c, tier, toks, 64, wf, role, 1.0, 1 if pin else 0)
            h = o.chain_hashes(toks)[0]
            d = o.dump(c, None, tier)
            bid = int(d["id"][d["hash"] == h][0])
            placed.append((bid, tier, wf, role, pin))
        before = {L1: o.dump(c, None, L1), L2: o.dump(c, None, L2)}
        o.complete(c, l3, 0, future, 2.0)
        after = {L1: set(o.dump(c, None, L1)["id"].tolist()),
                 L2: set(o.dump(c, None, L2)["id"].tolist())}
        l3ids = o.dump(c, l3, L3)
        for bid, tier, wf, role, pin in placed:
            if pin or wf != 0:
                assert bid in after[tier]
            elif (future >> role) & 1:
                assert bid in after[tier]
                h = before[tier]["hash"][before[tier]["id"] == bid][0]
                assert h in l3ids["hash"]
            else:
                assert bid not in after[tier]


# ---------------------------------------------------- test_cache.cpp eviction
def _reg(o):
    r = o.new_registry()
    o.reg_update(r, 0, 1 << 1)  # w_live=0 -> {"b"=1}
    return r


def test_evict_dead_before_live(be64):
    o = be64  # :284-294  roles b=1 dead=2
    r = _reg(o)
    c = o.new_cache(128, 10000)
    o.insert_chain(c, L1, make_tokens(1, 64), 64, 0, 1, 5.0, 0)
    o.insert_chain(c, L1, make_tokens(2, 64), 64, 0, 2, 9.0, 0)
    ok, ids, ft = o.evict_ids(c, L1, 64, r, True)
    assert ok and len(ids) == 1
    d = o.dump(c, None, L1)
    assert len(d) == 1 and d["role"][0] == 1


def test_evict_all_dead_oldest_first(be64):
    o = be64  # :295-303 wf x=5
    r = _reg(o)
    c = o.new_cache(192, 10000)
    for salt, t in ((1, 3.0), (2, 1.0), (3, 2.0)):
        o.insert_chain(c, L1, make_tokens(salt, 64), 64, 5, 0, t, 0)
    ok, ids, ft = o.evict_ids(c, L1, 128, r, True)
    assert len(ids) == 2
    assert o.dump(c, None, L1)["la"][0] == 3.0


def test_evict_two_phase_sort_oracle_seed11(be64):
    o = be64  # :304-350
    r = _reg(o)
    rng = MT19937_64(11)
    for trial in range(100):
        c = o.new_cache(100000, 10000)
        items = []
        occ = 0
        for i in range(15):
            dead = rng() % 2
            pin = rng() % 5 == 0
            access = float(rng() % 100)
            toks = make_tokens(5000 + trial * 100 + i, 64)
            o.insert_chain(c, L1, toks, 64, 1 if dead else 0, 1, access, 1 if pin else 0)
            h = o.chain_hashes(toks)[0]
            d = o.dump(c, None, L1)
            items.append((int(d["id"][d["hash"] == h][0]), bool(dead), pin, access, 64))
            occ += 64
        needed = 100000 - occ + rng() % 500
        ok, ids, ft = o.evict_ids(c, L1, needed, r, True)
        cand = sorted([x for x in items if not x[2]], key=lambda x: (not x[1], x[3], x[0]))
        excess = occ + needed - 100000
        expect, freed = [], 0
        for x in cand:
            if freed >= excess:
                break
            expect.append(x[0])
            freed += x[4]
        assert ids.tolist() == expect


def test_evict_speculative_off_is_lru(be64):
    o = be64  # :351-359
    r = _reg(o)
    c = o.new_cache(128, 10000)
    o.insert_chain(c, L1, make_tokens(1, 64), 64, 0, 1, 1.0, 0)
    o.insert_chain(c, L1, make_tokens(2, 64), 64, 0, 2, 9.0, 0)
    ok, ids, ft = o.evict_ids(c, L1, 64, r, False)
    assert len(ids) == 1
    assert o.dump(c, None, L1)["la"][0] == 9.0


def test_evict_insufficient(be64):
    o = be64  # :360-366
    r = _reg(o)
    c = o.new_cache(128, 10000)
    o.insert_chain(c, L1, make_tokens(1, 64), 64, 5, 0, 1.0, 1)
    o.insert_chain(c, L1, make_tokens(2, 64), 64, 5, 0, 1.0, 1)
    ok, ids, ft = o.evict_ids(c, L1, 64, r, True)
    assert not ok


# ------------------------------------------------------ test_sched.cpp routes
def _nodes(spec):
    """spec: list of (id, cap, [ (prompt, upper, alpha, gen), ...], staged)"""
    rid = [s[0] for s in spec]
    cap = [s[1] for s in spec]
    off = [0]
    asg = []
    for s in spec:
        asg.extend(s[2])
        off.append(len(asg))
    staged = [s[3] for s in spec]
    return rid, cap, off, np.array(asg, dtype=[("prompt_len", "<i8"), ("upper", "<i8"),
                                               ("alpha", "<f8"), ("tokens_generated", "<i8")]), staged


def route(o, spec, req, eps=0.05):
    rid, cap, off, asg, staged = _nodes(spec)
    return o.route(rid, cap, off, asg, staged, req, eps)


def test_route_kats(be64):
    o = be64
    req = (0, 100, 0.01, 0)  # test_sched.cpp:63-98
    t, tb, hr, ob = route(o, [(7, 1000, [], 0)], req)
    assert (t, hr) == (7, 900) and abs(ob - 0.01) < 1e-12
    t, tb, hr, ob = route(o, [(1, 1000, [(0, 400, 0.0, 0)], 0), (2, 1000, [(0, 600, 0.0, 0)], 0)],
                          req)
    assert t == 1 and tb == 0
    t, tb, _, _ = route(o, [(1, 1000, [], 0), (2, 1000, [], 400)], req)
    assert t == 2 and tb == 1
    t, _, _, _ = route(o, [(4, 1000, [], 0), (3, 1000, [], 0)], req)
    assert t == 3
    assert route(o, [(1, 1000, [(0, 950, 0.0, 0)], 0)], req)[0] == -1
    assert route(o, [(1, 10000, [(0, 10, 0.04, 0), (0, 10, 0.04, 0)], 0)], req)[0] == -1


def test_route_alpha_trap_kmax4(be64):
    """alpha = 1-0.99 = 0.010000000000000009; five of them sum above 0.05."""
    o = be64
    a = 1 - 0.99
    req = (10, 10, a, 0)
    for k in range(6):
        t = route(o, [(0, 10**9, [(10, 10, a, 0)] * k, 0)], req)[0]
        assert (t == 0) == (k + 1 <= 4)


def test_route_safety_seed5(be64):
    o = be64  # test_sched.cpp:100-123
    rng = MT19937_64(5)
    for _ in range(500):
        spec = []
        n = 1 + rng() % 5
        for i in range(n):
            cap = 2000 + rng() % 2000
            k = rng() % 6
            asg = []
            for j in range(k):
                p = rng() % 200
                u = rng() % 500
                al = 0.005 * float(rng() % 5)
                asg.append((p, u, al, 0))
            spec.append((i, cap, asg, 0))
        p = rng() % 200
        u = rng() % 500
        req = (p, u, 0.01, 0)
        t, tb, hr, ob = route(o, spec, req)
        if t >= 0:
            node = spec[t]
            tot = p + u + sum(a[0] + max(a[1], a[3]) for a in node[2])
            assert tot <= node[1]
            s = 0.01
            for a in node[2]:
                s += a[2]
            assert s <= 0.05 and ob == s


def test_route_least_outstanding(be64):
    # test_sched.cpp:125-130
    assert be64.route_least_outstanding([1, 2], [0, 2, 3]) == 2


# ------------------------------------------- differential: restated vs reference
need_ref16 = pytest.mark.skipif(not reference_available(16), reason="oracle/_ref not built")


def _random_ops(o, seed, B, n_ops=400):
    """A random op stream over one replica + L3; returns a transcript of every output."""
    rng = np.random.default_rng(seed)
    c, l3, reg = o.new_cache(int(rng.integers(200, 3000)), int(rng.integers(200, 3000))), \
        o.new_l3(), o.new_registry()
    bases = [rng.integers(0, 1 << 62, size=400, dtype=np.uint64) for _ in range(4)]
    out = []
    now = 0.0
    for step in range(n_ops):
        now += float(rng.integers(0, 3))
        base = bases[int(rng.integers(0, 4))]
        n = int(rng.integers(0, 300))
        toks = base[:n].copy()
        if n and rng.random() < 0.3:
            toks[int(rng.integers(0, n))] ^= np.uint64(1)
        op = rng.random()
        wf, role = int(rng.integers(0, 6)), int(rng.integers(0, 5))
        if op < 0.25:
            tier = int(rng.integers(0, 2))
            upto = int(rng.integers(0, n + 1)) if rng.random() < 0.3 else n
            pin = int(rng.integers(-1, 3))
            o.insert_chain(c, tier, toks, upto, wf, role, now, pin)
            out.append(("ins",))
        elif op < 0.45:
            out.append(("lk", o.lookup(c, l3, toks)))
        elif op < 0.55:
            o.unpin_chain(c, toks, n)
            out.append(("unpin",))
        elif op < 0.68:
            for w in range(6):
                if rng.random() < 0.5:
                    o.reg_update(reg, w, int(rng.integers(0, 32)))
                elif rng.random() < 0.2:
                    o.reg_drop(reg, w)
            tier = int(rng.integers(0, 2))
            ok, ids, ft = o.evict_ids(c, tier, int(rng.integers(0, 400)), reg,
                                      bool(rng.integers(0, 2)))
            out.append(("ev", ok, ids.tolist(), ft))
        elif op < 0.76:
            m = int(rng.integers(0, 32))
            out.append(("cmp", o.complete(c, l3, wf, m, now)))
            o.l3_dead_sweep(l3, wf, m)
        elif op < 0.84:
            tier = int(rng.integers(0, 3))
            frm = int(rng.integers(0, n + 1))
            o.erase_chain_span(c, l3, tier, toks, frm, int(rng.integers(frm, n + 1)))
            out.append(("span",))
        elif op < 0.9:
            o.add_decode(c, int(rng.integers(-50, 100)))
            out.append(("dec", o.l1_occupancy(c)))
        else:
            tier = int(rng.integers(0, 3))
            h = int(o.chain_hashes(toks)[-1]) if n else int(rng.integers(0, 1 << 62))
            s = int(rng.integers(0, 4)) * B
            e = s + int(rng.integers(1, 2 * B))
            out.append(("put", o.put(c, l3, tier, h, s, e, wf, role, now, int(rng.integers(0, 2)))))
            d = o.dump(c, l3, tier)
            if len(d) and rng.random() < 0.5:
                o.erase(c, l3, tier, int(d["id"][int(rng.integers(0, len(d)))]))
        for tier in (L1, L2, L3):
            d = o.dump(c, l3 if tier == L3 else None, tier)
            out.append((tier, d.tobytes()))
    return out


@need_ref16
@pytest.mark.parametrize("B", [16, 64])
@pytest.mark.parametrize("seed", range(6))
def test_restated_equals_reference_random_ops(B, seed):
    if not reference_available(B):
        pytest.skip("no reference build")
    a = _random_ops(Restated(B), seed, B)
    b = _random_ops(Reference(B), seed, B)
    assert len(a) == len(b)
    for i, (x, y) in enumerate(zip(a, b)):
        assert x == y, f"op {i}: {x} vs {y}"


@need_ref16
@pytest.mark.parametrize("seed", range(4))
def test_restated_route_equals_reference_random(seed):
    o, r = Restated(16), Reference(16)
    rng = np.random.default_rng(1000 + seed)
    for _ in range(2000):
        n = int(rng.integers(1, 12))
        spec = []
        for i in rng.permutation(n):
            k = int(rng.integers(0, 7))
            asg = [(int(rng.integers(0, 50)), int(rng.integers(0, 50)),
                    float(rng.choice([0.0, 1 - 0.99, 0.005, 0.02])), int(rng.integers(0, 80)))
                   for _ in range(k)]
            spec.append((int(i), int(rng.integers(100, 400)), asg, int(rng.integers(0, 3))))
        req = (int(rng.integers(0, 50)), int(rng.integers(0, 50)),
               float(rng.choice([0.0, 1 - 0.99])), int(rng.integers(0, 60)))
        assert route(o, spec, req) == route(r, spec, req)
