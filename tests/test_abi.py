"""The C-ABI library loads and exports every symbol include/pyg.h declares (CPU: no
compute calls); without a GPU pyg_create fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "pyg.h")).read()
    return sorted(set(re.findall(r"^(?:int|void|const char\*|int64_t)\s+(pyg_\w+)\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ["pyg_create", "pyg_lookup", "pyg_insert_chain", "pyg_evict_for_space",
                 "pyg_route", "pyg_complete", "pyg_hash_batch_dev", "pyg_route_batch_dev",
                 "pyg_admit_batch_dev", "pyg_step_host"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2604_25899_b200 import _lib
    lib = ctypes.CDLL(_lib.SO_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2604_25899_b200 import Context, PygError
    with pytest.raises(PygError) as e:
        Context(1, 100, 100, 16)
    assert "ECUDA" in str(e.value)


def test_so_is_sm100a():
    from paper_2604_25899_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", _lib.SO_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
