"""The C-ABI library loads without a GPU and exports exactly what
include/cvgram_b200.h declares (no compute calls here)."""
import ctypes
import os
import re

from paper_2401_13185_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "cvgram_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cvg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_abi():
    names = declared()
    assert "cvg_run_all_folds" in names and "cvg_plan_finish" in names and len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert sorted(_lib.SIGNATURES) == declared()


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        return
    from paper_2401_13185_b200 import cvgram as cv

    try:
        cv.Context(0)
    except cv.DeviceError as e:
        assert "no CUDA device" in str(e)
    else:
        raise AssertionError("context creation must fail without a device")
