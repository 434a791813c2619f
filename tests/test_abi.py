"""The C-ABI library loads and exports every entry point include/tinv.h declares.
No compute calls (runs without a GPU)."""
import ctypes as C
import os
import re

import pytest

from paper_1209_1910_b200 import tinv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "tinv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tinv_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_api():
    names = declared_functions()
    for required in ("tinv_create", "tinv_eigvecs", "tinv_destroy", "tinv_strerror"):
        assert required in names
    assert set(names) == set(tinv.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = tinv.load_library()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert L.tinv_abi_version() == 1
    assert L.tinv_strerror(0) == b"success"
    assert b"ldz" in L.tinv_strerror(-7)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {tinv.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    L = tinv.load_library()
    h = C.c_void_p()
    cfg = tinv.TinvConfig(0, 1, 0, None, None)
    assert L.tinv_create(C.byref(h), C.byref(cfg)) == -100
    with pytest.raises(tinv.TinvError):
        tinv.Tinv(0)


def test_product_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_1209_1910_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "liboracle" not in txt, f
