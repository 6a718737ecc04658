"""CPU-only checks of the drop-in boundary: the C-ABI library builds/loads and
exports every entry point include/zsort_b200.h declares (no compute calls)."""

import ctypes
import os
import re

import pytest

from paper_2605_14419_b200 import _lib, build

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(REPO, "include", "zsort_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(zsb_[a-z_0-9]+)\s*\(", txt)))


def test_library_builds_and_loads():
    path = build.build()
    assert os.path.exists(path)
    L = _lib.load()
    assert b"sm_100a" in L.zsb_version()


def test_every_declared_symbol_is_exported():
    L = ctypes.CDLL(build.LIB)
    declared = header_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.EXPORTS)


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_workspace_bytes_grow_with_n():
    L = _lib.load()
    a = L.zsb_workspace_bytes(10**6, 0, 4, None)
    b = L.zsb_workspace_bytes(10**7, 0, 4, None)
    c = L.zsb_workspace_bytes(10**7, 0, 8, None)
    assert 12 * 10**6 < a < b < c
    assert b >= 12 * 10**7  # scratch keys + payload


def test_config_validation_mirrors_reference():
    from paper_2605_14419_b200 import SortConfig
    with pytest.raises(ValueError):
        SortConfig(alpha=0)
    with pytest.raises(ValueError):
        SortConfig(alpha=2.5)
    with pytest.raises(ValueError):
        SortConfig(insertion_threshold=0)
    with pytest.raises(ValueError):
        SortConfig(counting_range_threshold=0)
    with pytest.raises(ValueError):
        SortConfig(depth_guard=2)
    with pytest.raises(ValueError):
        SortConfig(mapping="radix")
    SortConfig(alpha=2.0, depth_guard=3, mapping="paper")


def test_dtype_gate_without_gpu():
    import numpy as np
    from paper_2605_14419_b200 import zsort
    with pytest.raises(TypeError):
        zsort(np.array([1, 2], np.uint64))
    with pytest.raises(TypeError):
        zsort(np.array([1.5, 2.5], np.float32))
    with pytest.raises(ValueError):
        zsort(np.zeros((2, 2), np.int64))
    with pytest.raises(ValueError):
        zsort(np.array([1, 2], np.int64), payload=np.arange(3))
    k, p, s = zsort(np.array([], np.int64))
    assert k.size == 0 and p is None and s.total_scatter_passes == 0
