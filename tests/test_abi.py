"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/csc.h declares.
No compute calls here (no GPU in this container)."""
import os
import re
import subprocess

import pytest

import paper_1909_00145_b200 as pkg
from paper_1909_00145_b200 import build as b

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    b.build()
    return pkg.load_library()


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "csc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(csc_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert sorted(pkg.ABI_SYMBOLS) == _declared_symbols()


def test_library_exports_every_declared_symbol(lib):
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", pkg.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (csc_[a-z0-9_]+)\b", out))
    assert set(_declared_symbols()) <= exported


def test_abi_version(lib):
    assert lib.csc_abi_version() == 1


def test_sm100a_cubin_embedded():
    out = subprocess.run(["cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_init_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import ctypes
    dims = pkg._Dims(1, 2, 3, 8, 8, 1, 0, 0, None, None)
    h = ctypes.c_void_p()
    st = lib.csc_init(ctypes.byref(dims), ctypes.byref(h))
    assert st == 3  # CSC_ERR_CUDA: no CPU fallback
    assert b"CUDA" in lib.csc_last_error(None) or b"device" in lib.csc_last_error(None)


def test_init_argument_validation(lib):
    import ctypes
    for bad in [(1, 0, 3, 8, 8), (1, 2, 4, 8, 8), (1, 2, 5, 4, 8), (-1, 2, 3, 8, 8)]:
        dims = pkg._Dims(*bad, 1, 0, 0, None, None)
        h = ctypes.c_void_p()
        assert lib.csc_init(ctypes.byref(dims), ctypes.byref(h)) == 1  # CSC_ERR_ARG before touching CUDA
    dims = pkg._Dims(1, 2, 3, 8, 8, 3, 0, 0, None, None)
    assert lib.csc_init(ctypes.byref(dims), ctypes.byref(ctypes.c_void_p())) == 1


def test_product_path_does_not_import_oracle():
    """The product package never references the oracle (it must fail loudly, never fall back)."""
    pkgdir = os.path.join(ROOT, "paper_1909_00145_b200")
    for dirpath, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "oracle." not in txt, f
