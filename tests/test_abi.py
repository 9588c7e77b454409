"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol
include/nmg.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2603_01064_b200 as nmg
from paper_2603_01064_b200 import binding, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "nmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nmg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return binding.load_library()


def test_header_declares_the_boundary():
    syms = _declared_symbols()
    for s in ("nmg_create_hierarchy", "nmg_load_smoother_weights", "nmg_vcycle", "nmg_solve"):
        assert s in syms
    assert set(binding.EXPORTS) == set(syms)


def test_library_exports_every_declared_symbol(lib):
    for s in _declared_symbols():
        assert hasattr(lib, s), s
    assert lib.nmg_version().decode().startswith("nmg-b200")


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", binding.lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_error_not_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(nmg.NmgError) as ei:
        nmg.Hierarchy(1, 16, 2, 1e-2, [np.eye(16)], max_rhs=1)
    assert ei.value.status == 6          # NMG_ERR_CUDA
    assert "no CPU fallback" in str(ei.value)


def test_invalid_arguments_rejected(lib):
    with pytest.raises(nmg.NmgError) as ei:
        nmg.Hierarchy(1, 12, 2, 1e-2, [np.eye(12)], max_rhs=1)     # not a power of two
    assert ei.value.status == 1
    with pytest.raises(nmg.NmgError) as ei:
        nmg.Hierarchy(1, 16, 2, -1.0, [np.eye(16)], max_rhs=1)
    assert ei.value.status == 1
    with pytest.raises(nmg.NmgError) as ei:
        nmg.Hierarchy(3, 16, 2, 1.0, [np.eye(16)], max_rhs=1)
    assert ei.value.status == 1
