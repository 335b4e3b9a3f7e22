"""bench.py's argument contract (CPU): the K1 overlap defaults resolve per GPU count, the
workload defaults fill in, and the reference arm's flags parse."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _parse(argv, world=None, monkeypatch=None):
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py", *argv])
    if world is None:
        monkeypatch.delenv("WORLD_SIZE", raising=False)
    else:
        monkeypatch.setenv("WORLD_SIZE", str(world))
    return bench.parse()


def test_auto_overlap_one_gpu(monkeypatch):
    a = _parse([], monkeypatch=monkeypatch)
    assert (a.k1_grid, a.k1_after) == ("tasks1", "start")
    assert a.workload == "bursty" and a.requests == 125_000 and a.replicas == 256


@pytest.mark.parametrize("argv,world", [(["--gpus", "4"], None), (["--gpus", "2"], "2"),
                                        ([], "8")])
def test_auto_overlap_several_gpus(argv, world, monkeypatch):
    a = _parse(argv, world, monkeypatch)
    assert (a.k1_grid, a.k1_after) == ("tasks1", "staged")


def test_explicit_overlap_kept(monkeypatch):
    a = _parse(["--gpus", "2", "--k1-grid", "tasks1", "--k1-after", "start"],
               monkeypatch=monkeypatch)
    assert (a.k1_grid, a.k1_after) == ("tasks1", "start")


def test_auto_overlap_config3(monkeypatch):
    a = _parse(["--workload", "long_context"], monkeypatch=monkeypatch)
    assert (a.k1_grid, a.k1_after, a.free_sms) == ("persistent", "start", 48)
    a = _parse([], monkeypatch=monkeypatch)
    assert a.free_sms == 8


def test_reference_arm_and_config3(monkeypatch):
    a = _parse(["--impl", "reference", "--workload", "long_context", "--steps", "2",
                "--warmup", "3"], monkeypatch=monkeypatch)
    assert a.impl == "reference" and a.workload == "long_context"
    assert a.steps == 2 and a.warmup == 3
