"""ctypes binding of the C ABI in include/cvgram_b200.h.

The shared library is built in-tree (``paper_2401_13185_b200/_build``) by
``__graft_entry__.build()``.  There is deliberately no fallback: if the library
is missing, importing the compute API raises, and without an sm_100 device
every compute call fails with CVG_E_CUDA.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CVG_LIB_VARIANT=checked loads the bounds-checked build (make CHECKED=1 -> _build_checked/);
# any other name loads _build_<name>/ (make OUT=_build_<name> EXTRA=-D...: experiment builds).
_VARIANT = os.environ.get("CVG_LIB_VARIANT", "")
LIB_PATH = os.path.join(_HERE, f"_build_{_VARIANT}" if _VARIANT else "_build", "libcvgram_b200.so")

OK, E_DIMENSION, E_PARTITION, E_SCALABILITY, E_INVALID_ARG, E_CUDA, E_OOM, E_NCCL = 0, 1, 2, 3, 4, 5, 6, 7
DTYPE_F64, DTYPE_F32 = 0, 1

c_i64, c_i32, c_u32, c_u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64
c_vp, c_char_p, c_size_t, c_int, c_double = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_double
c_vpp = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); mirrors include/cvgram_b200.h one to one.
SIGNATURES = {
    "cvg_version": (c_int, []),
    "cvg_context_create": (c_int, [c_int, c_vpp, c_char_p, c_size_t]),
    "cvg_context_destroy": (None, [c_vp]),
    "cvg_context_set_stream": (c_int, [c_vp, c_vp]),
    "cvg_context_launch_count": (c_i64, [c_vp]),
    "cvg_context_enable_timing": (c_int, [c_vp, c_int]),
    "cvg_context_kernel_times": (c_int, [c_vp, c_vp, c_vp]),
    "cvg_validate_dataset": (c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_char_p, c_size_t]),
    "cvg_validate_partitioning": (c_int, [c_vp, c_i64, c_i32, c_char_p, c_size_t]),
    "cvg_check_scalable": (c_int, [c_vp, c_i64, c_i32, c_char_p, c_size_t]),
    "cvg_fold_range": (c_int, [c_i32, c_i32, c_i32, c_vp, c_vp]),
    "cvg_run_all_folds": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i32, c_vp, c_i32]
                          + [c_vp] * 8 + [c_char_p, c_size_t]),
    "cvg_plan_create": (c_int, [c_vp, c_int, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_vpp, c_char_p, c_size_t]),
    "cvg_plan_create_rank": (c_int, [c_vp, c_int, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_vpp, c_char_p,
                                     c_size_t]),
    "cvg_plan_assignment": (c_int, [c_vp, c_vp, c_vp]),
    "cvg_plan_destroy": (None, [c_vp]),
    "cvg_plan_bind_labels": (c_int, [c_vp, c_vp, c_int, c_char_p, c_size_t]),
    "cvg_plan_gram": (c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_char_p, c_size_t]),
    "cvg_plan_gram_mapped": (c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_char_p, c_size_t]),
    "cvg_run_all_folds_stream": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i32, c_vp, c_i32,
                                         c_i32, c_vp, c_vp, c_char_p, c_size_t]),
    "cvg_plan_finish_range": (c_int, [c_vp, c_vp, c_i32, c_vp, c_i32, c_i32, c_i32] + [c_vp] * 6 + [c_char_p, c_size_t]),
    "cvg_plan_partial": (c_int, [c_vp, c_vp, ctypes.POINTER(c_i64)]),
    "cvg_plan_finish": (c_int, [c_vp, c_vp, c_i32, c_vp, c_i32] + [c_vp] * 6 + [c_char_p, c_size_t]),
    "cvg_plan_fold_counts": (c_int, [c_vp, c_vp]),
    "cvg_global_create": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_i64, c_i64, c_vpp, c_char_p, c_size_t]),
    "cvg_global_destroy": (None, [c_vp]),
    "cvg_global_export": (c_int, [c_vp, c_u32] + [c_vp] * 8 + [c_char_p, c_size_t]),
    "cvg_global_fold_products": (c_int, [c_vp, c_vp, c_i64, c_u32] + [c_vp] * 7 + [c_char_p, c_size_t]),
    "cvg_baseline_fold_products": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i32, c_vp,
                                           c_i32] + [c_vp] * 8 + [c_char_p, c_size_t]),
    "cvg_baseline_single_fold": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_u32] + [c_vp] * 7
                                 + [c_char_p, c_size_t]),
    "cvg_rng_create": (c_vp, [c_u64]),
    "cvg_rng_destroy": (None, [c_vp]),
    "cvg_rng_next": (c_u64, [c_vp]),
    "cvg_rng_uniform01": (c_double, [c_vp]),
    "cvg_random_dataset": (None, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "cvg_random_partitioning": (None, [c_vp, c_i64, c_i32, c_vp]),
    "cvg_uniform01_bits": (c_double, [c_u64]),
    "cvg_random_dataset_fn": (None, [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "cvg_random_partitioning_fn": (None, [c_vp, c_vp, c_i64, c_i32, c_vp]),
    "cvg_training_mean": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_char_p, c_size_t]),
    "cvg_training_std": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_char_p, c_size_t]),
    "cvg_hadamard_outer_divide": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_char_p,
                                          c_size_t]),
    "cvg_selftest_division": (c_int, [c_vp, c_i64, c_u64, c_vp, c_vp]),
    "cvg_context_create_multi": (c_int, [c_int, c_vp, c_vp, c_char_p, c_size_t]),
    "cvg_context_device_count": (c_int, [c_vp]),
    "cvg_context_exchange": (c_int, [c_vp]),
    "cvg_host_alloc": (c_int, [c_size_t, c_vp]),
    "cvg_host_free": (None, [c_vp]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load the engine library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"cvgram B200 engine library missing at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def err_buf():
    return ctypes.create_string_buffer(1024)
