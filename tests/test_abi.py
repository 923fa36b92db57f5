"""C-ABI checks that need no GPU (-m "not gpu"): the library builds, loads and
exports every symbol include/gbla.h declares; without a GPU it refuses to
run (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gbla.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gbla_[A-Za-z_0-9]+)\s*\(", src)) - {"gbla_alloc_fn", "gbla_free_fn", "gbla_memq_fn"})


@pytest.fixture(scope="module")
def lib():
    from paper_1602_06097_b200 import build as b
    path = b.build()
    return ctypes.CDLL(path)


def test_header_declares_the_six_calls():
    d = _declared()
    for name in ("gbla_splice", "gbla_reduce_B", "gbla_reduce_C", "gbla_update_D", "gbla_echelon_D", "gbla_reduce"):
        assert name in d


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1602_06097_b200", "libgbla.so")],
                         capture_output=True, text=True).stdout
    for s in _declared():
        assert re.search(rf"\sT\s{s}$", out, re.M), s


def test_binding_names_match_header():
    import paper_1602_06097_b200 as gb
    assert set(gb.exported_symbols()) <= set(_declared())
    for name in ("gbla_splice", "gbla_reduce_B", "gbla_reduce_C", "gbla_update_D", "gbla_echelon_D", "gbla_reduce"):
        assert callable(getattr(gb, name))


def test_library_is_sm100a_code(lib):
    so = os.path.join(ROOT, "paper_1602_06097_b200", "libgbla.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_error_not_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib.gbla_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    h = ctypes.c_void_p()
    assert lib.gbla_ctx_create(0, ctypes.byref(h)) == 5          # GBLA_E_CUDA
    lib.gbla_last_error.restype = ctypes.c_char_p
    assert b"no CUDA device" in lib.gbla_last_error()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1602_06097_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gbla_oracle" not in txt and "liboracle" not in txt, f
