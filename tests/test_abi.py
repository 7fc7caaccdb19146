"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads,
and exports every function include/tem_b200.h declares; the binding refuses
CPU tensors (no fallback).  No compute calls (there is no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tem_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tem_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_11657_b200 import _lib, build
    build.build()
    return _lib.load()


def test_header_declares_expected_calls():
    names = _declared()
    for must in ("tem_create", "tem_edge_mass", "tem_apply_shifted", "tem_cocg_solve",
                 "tem_synthesize", "tem_forward_host"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2506_11657_b200 import build
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tem_[a-z_]+)\b", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    for n in _declared():
        assert hasattr(lib, n)


def test_library_is_sm100a(lib):
    from paper_2506_11657_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string(lib):
    assert lib.tem_version().decode().startswith("tem_b200")
    assert isinstance(lib.tem_last_error(), bytes)


def test_invalid_arguments_rejected_before_launch(lib):
    import ctypes
    import numpy as np
    h = ctypes.c_void_p()
    hx = np.ones(1)
    dp = hx.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    assert lib.tem_create(1, 4, 4, dp, dp, dp, ctypes.byref(h)) == -1     # nx < 2
    assert b"nx" in lib.tem_last_error()
    neg = np.array([1.0, -2.0])
    dn = neg.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    assert lib.tem_create(2, 2, 2, dn, dn, dn, ctypes.byref(h)) == -1     # h <= 0
    assert lib.tem_cocg_workspace_bytes(None, 4) == 0


def test_solver_selection_argument_checks(lib):
    # NULL context: rejected before any CUDA call
    assert lib.tem_set_solver(None, 0) == -1
    assert lib.tem_get_solver(None) == -1
    assert b"tem_set_solver" in lib.tem_last_error()


def test_binding_refuses_cpu_tensors():
    import torch
    from paper_2506_11657_b200.solver import _need_cuda
    with pytest.raises(ValueError):
        _need_cuda(torch.zeros(3, dtype=torch.float64), torch.float64, "sigma")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2506_11657_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", txt, flags=re.M), fn
                assert "oracle/" not in txt.replace("never imports the CPU oracle", ""), fn
