"""CPU: the C-ABI library builds, loads and exports exactly what
include/idkit_b200.h declares; without a GPU every entry fails loudly
(IDK_ERR_CUDA) -- there is no CPU fallback.  No compute runs here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "idkit_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"IDK_API\s+[\w\s\*]+?\b(idk_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2105_07076_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2105_07076_b200 import build
        build.build()
    return _lib


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("idk_optim_id", "idk_sketch_rid", "idk_id_auto", "idk_optim_id_batched", "idk_id_from_sketch",
              "idk_qr_column_pivoted", "idk_select_columns", "idk_sketch", "idk_sketch_omega", "idk_id_auto_host"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r" T (idk_\w+)", out.stdout))
    assert set(declared_symbols()) <= exported
    assert exported <= set(declared_symbols()), "exports not declared in the header"


def test_ctypes_signatures_cover_header(lib):
    assert set(lib.SIGNATURES) == set(declared_symbols())
    L = lib.load()
    for name in lib.SIGNATURES:
        assert hasattr(L, name)
    assert L.idk_abi_version() == 1


def test_kernels_are_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True,
                         text=True, check=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    assert "DMMA" in sass  # the sketch GEMM runs on the FP64 tensor pipe


def test_status_strings(lib):
    L = lib.load()
    assert L.idk_status_string(0) == b"ok"
    assert L.idk_status_string(2) == b"singular matrix"
    assert L.idk_status_string(3) == b"not positive definite"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly(lib):
    L = lib.load()
    h = ctypes.c_void_p()
    assert L.idk_create(ctypes.byref(h), 0) == 4  # IDK_ERR_CUDA
    import paper_2105_07076_b200 as idk
    with pytest.raises(idk.CudaError):
        idk.Context(0)
    with pytest.raises(idk.CudaError):
        idk.id_auto(np.eye(4), 2)


def test_null_handle_is_invalid_argument(lib):
    L = lib.load()
    assert L.idk_optim_id(None, None, 4, 4, 4, 2, None, None, None) == 1
    assert L.idk_sketch_rid(None, None, 4, 4, 4, 0, 2, 1, 0, 0, None, None, None, None) == 1


def test_missing_library_raises(tmp_path):
    from paper_2105_07076_b200 import _lib
    with pytest.raises(_lib.IdkitLibraryMissing):
        _lib.load(str(tmp_path / "nope.so"))
