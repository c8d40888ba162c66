"""CPU-side checks of the boundary: the C-ABI library builds/loads without a GPU
and exports every symbol include/srk.h declares; the product path refuses to
run without CUDA (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "srk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(srk_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for need in ("srk_solve", "srk_spmm_block", "srk_gram_block", "srk_block_update", "srk_tsqr",
                 "srk_matrix_create", "srk_create"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    import paper_1504_04395_b200 as srk
    if not os.path.exists(srk._LIBPATH):
        from paper_1504_04395_b200 import build
        build.build(verbose=False)
    lib = ctypes.CDLL(srk._LIBPATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(srk.EXPORTS) <= set(declared_symbols())
    assert lib.srk_version() == 1


def test_no_cpu_fallback():
    import torch
    import paper_1504_04395_b200 as srk
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    srk.load_library()
    with pytest.raises(srk.SrkError):
        srk.Context()
    lib = srk.load_library()
    h = ctypes.c_void_p()
    assert lib.srk_create(ctypes.byref(h), 0, None) == -4  # SRK_ECUDA
    assert b"srk_create" in lib.srk_last_error()


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1504_04395_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "oracle/" not in txt or f.endswith((".cu", ".cuh", ".h")), f
