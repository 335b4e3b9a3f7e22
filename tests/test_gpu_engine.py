"""Whole-trace parity through the drop-in boundary: the reference's
own simulator engine (src/sim/engine.cpp, unmodified) is built twice -- with the reference
cache/router (oracle/_ref/engine_ref16) and with the B200 backend behind the same C++
interfaces (integration/_build/engine_b200, integration/pyg_adapter.cpp).  On the built-in
coding-assistant workload both must write byte-identical event, routing, cache-action and
scaling logs and metrics.  The binaries are built where /root/reference exists
(__graft_entry__.build()); the test skips when they are absent."""
import filecmp
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "engine_ref16")
B200 = os.path.join(ROOT, "integration", "_build", "engine_b200")
FILES = ["event_log.txt", "routing_log.jsonl", "cache_log.jsonl", "scale_log.jsonl",
         "metrics.json"]


@pytest.mark.parametrize("workflows,seed", [(20, 1), (12, 7)])
def test_reference_engine_on_b200_is_byte_identical(tmp_path, workflows, seed):
    if not (os.path.exists(REF) and os.path.exists(B200)):
        pytest.skip("engine binaries not built (need /root/reference at build time)")
    outs = {}
    for name, exe in (("ref", REF), ("b200", B200)):
        d = tmp_path / name
        d.mkdir()
        p = subprocess.run([exe, str(d), str(workflows), str(seed)], capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs[name] = d
    for f in FILES:
        a, b = outs["ref"] / f, outs["b200"] / f
        assert a.stat().st_size > 0, f
        assert filecmp.cmp(a, b, shallow=False), f"{f} differs"
    with open(outs["ref"] / "event_log.txt") as fh:
        assert sum(1 for _ in fh) > 100
