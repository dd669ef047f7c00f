"""ctypes bindings for the C oracle (test infrastructure only).

Every function cites the reference entity it restates; see cvgram_oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libcvgram_oracle.so")

OK, E_DIMENSION, E_PARTITION, E_SCALABILITY, E_INVALID_ARG, E_CUDA, E_OOM = 0, 1, 2, 3, 4, 5, 6
CX, CY, SX, SY = 8, 4, 2, 1

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


class OracleError(ValueError):
    """Raised with the reference's error code (core.hpp:20-32) and message."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_rng_new.restype = _vp
        L.orc_rng_new.argtypes = [ctypes.c_uint64]
        L.orc_rng_free.argtypes = [_vp]
        L.orc_rng_next.restype = ctypes.c_uint64
        L.orc_rng_next.argtypes = [_vp]
        L.orc_uniform01.restype = ctypes.c_double
        L.orc_uniform01.argtypes = [_vp]
        L.orc_random_dataset.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp]
        L.orc_random_partitioning.argtypes = [_vp, _i64, _i32, _vp]
        for name in ("orc_validate_partitioning", "orc_check_scalable"):
            getattr(L, name).argtypes = [_vp, _i64, _i32, ctypes.c_char_p, ctypes.c_size_t]
        L.orc_build_validation_partitions.argtypes = [_vp, _i64, _i32, _vp, _vp]
        L.orc_complement_rows.restype = _i64
        L.orc_complement_rows.argtypes = [_vp, _i64, _i64, _vp]
        L.orc_hadamard_outer_divide.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, ctypes.c_char_p,
                                                ctypes.c_size_t]
        L.orc_max_rel_diff.restype = ctypes.c_double
        L.orc_max_rel_diff.argtypes = [_vp, _vp, _i64, ctypes.c_double]
        L.orc_rel_frobenius_dist.restype = ctypes.c_double
        L.orc_rel_frobenius_dist.argtypes = [_vp, _vp, _i64, ctypes.c_double]
        L.orc_precompute_global.argtypes = [_vp, _vp, _i64, _i64, _i64, _u32] + [_vp] * 8 + [ctypes.c_int]
        L.orc_training_mean.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, ctypes.c_char_p, ctypes.c_size_t]
        L.orc_training_std.argtypes = [_vp, _vp, _vp, _i64, _i64, _vp, ctypes.c_char_p, ctypes.c_size_t]
        L.orc_fold_products.argtypes = ([_vp, _vp, _i64, _i64, _i64] + [_vp] * 8 + [_vp, _i64, _u32] + [_vp] * 7
                                        + [ctypes.c_char_p, ctypes.c_size_t])
        L.orc_baseline_single_fold.argtypes = ([_vp, _vp, _i64, _i64, _i64, _vp, _i64, _u32] + [_vp] * 7
                                               + [ctypes.c_char_p, ctypes.c_size_t])
        for name in ("orc_fast_all_folds", "orc_baseline_all_folds"):
            getattr(L, name).argtypes = ([_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i32, _u32, ctypes.c_int]
                                         + [_vp] * 8 + [ctypes.c_char_p, ctypes.c_size_t])
        L.orc_truth_all_folds_multi.argtypes = ([_vp, _vp, ctypes.c_int, _i64, _i64, _i64, _vp, _i64, _i32, _vp,
                                                 ctypes.c_int, ctypes.c_int] + [_vp] * 8
                                                + [ctypes.c_char_p, ctypes.c_size_t])
        L.orc_truth_all_folds.argtypes = ([_vp, _vp, ctypes.c_int, _i64, _i64, _i64, _vp, _i64, _i32, _u32,
                                           ctypes.c_int] + [_vp] * 8 + [ctypes.c_char_p, ctypes.c_size_t])
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _check(rc, err):
    if rc != OK:
        raise OracleError(rc, err.value.decode())


def cfg_mask(center_x=False, center_y=False, scale_x=False, scale_y=False) -> int:
    return (CX if center_x else 0) | (CY if center_y else 0) | (SX if scale_x else 0) | (SY if scale_y else 0)


def enumerate_configs():
    """combos.hpp:33-45: 4-bit counter over (cx, cy, sx, sy), all-off first."""
    return list(range(16))


# ---------------------------------------------------------------- random.hpp
class MT64:
    """std::mt19937_64 stream plus the reference's generators (random.hpp:14-55)."""

    def __init__(self, seed: int):
        self._h = lib().orc_rng_new(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rng_free(self._h)
            self._h = None

    def next(self) -> int:
        return lib().orc_rng_next(self._h)

    def uniform01(self) -> float:
        return lib().orc_uniform01(self._h)

    def random_dataset(self, n, k, m):
        x = np.empty((n, k), np.float64)
        y = np.empty((n, m), np.float64)
        lib().orc_random_dataset(self._h, n, k, m, _p(x), _p(y))
        return x, y

    def random_partitioning(self, n, p):
        labels = np.empty(n, np.int32)
        lib().orc_random_partitioning(self._h, n, p, _p(labels))
        return labels


# ------------------------------------------------------------- partition.hpp
def validate_partitioning(labels, p):
    labels = np.ascontiguousarray(labels, np.int32)
    err = ctypes.create_string_buffer(512)
    rc = lib().orc_validate_partitioning(_p(labels), labels.size, p, err, 512)
    return None if rc == OK else err.value.decode()


def check_scalable(labels, p):
    labels = np.ascontiguousarray(labels, np.int32)
    err = ctypes.create_string_buffer(512)
    rc = lib().orc_check_scalable(_p(labels), labels.size, p, err, 512)
    return None if rc == OK else err.value.decode()


def build_validation_partitions(labels, p):
    labels = np.ascontiguousarray(labels, np.int32)
    rows = np.empty(max(labels.size, 1), np.int64)
    offs = np.empty(p + 1, np.int64)
    lib().orc_build_validation_partitions(_p(labels), labels.size, p, _p(rows), _p(offs))
    return [rows[offs[f]:offs[f + 1]].copy() for f in range(p)]


def complement_rows(v_rows, n):
    v = np.ascontiguousarray(v_rows, np.int64)
    out = np.empty(max(n, 1), np.int64)
    nt = lib().orc_complement_rows(_p(v), v.size, n, _p(out))
    return out[:nt].copy()


# ------------------------------------------------------------------ core.hpp
def hadamard_outer_divide(mat, left, right):
    mat = np.ascontiguousarray(mat, np.float64)
    left = np.ascontiguousarray(left, np.float64)
    right = np.ascontiguousarray(right, np.float64)
    out = np.empty_like(mat)
    err = ctypes.create_string_buffer(512)
    _check(lib().orc_hadamard_outer_divide(_p(mat), mat.shape[0], mat.shape[1], _p(left), left.size, _p(right),
                                           right.size, _p(out), err, 512), err)
    return out


def max_rel_diff(a, b, floor=1e-30):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if a.shape != b.shape:
        raise OracleError(E_DIMENSION, "max_rel_diff: shape mismatch")
    return lib().orc_max_rel_diff(_p(a), _p(b), a.size, floor)


def rel_frobenius_dist(a, b, floor=1e-30):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().orc_rel_frobenius_dist(_p(a), _p(b), a.size, floor)


# ------------------------------------------------------------------ fast.hpp
@dataclass
class Cache:
    xtx: np.ndarray
    xty: np.ndarray
    sum_x: np.ndarray
    sum_y: np.ndarray
    mean_x: np.ndarray
    mean_y: np.ndarray
    sum_sq_x: np.ndarray
    sum_sq_y: np.ndarray
    n_rows: int
    cfg: int


def precompute_global(x, y, cfg, n_threads=1) -> Cache:
    """fast.hpp:19-36 (unused vectors come back empty, as in the reference)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    n, k = x.shape
    m = y.shape[1]
    xtx = np.empty((k, k))
    xty = np.empty((k, m))
    v = [np.zeros(k), np.zeros(m), np.zeros(k), np.zeros(m), np.zeros(k), np.zeros(m)]
    lib().orc_precompute_global(_p(x), _p(y), n, k, m, cfg, _p(xtx), _p(xty), *[_p(a) for a in v], n_threads)
    e = np.empty(0)
    anyc = cfg & 15
    anys = cfg & (SX | SY)
    return Cache(xtx, xty, v[0] if anyc else e, v[1] if anyc else e, v[2] if anyc else e, v[3] if anyc else e,
                 v[4] if anys else e, v[5] if anys else e, n, cfg)


def training_mean(g, v, n, n_val):
    """fast.hpp:40-47."""
    g = np.ascontiguousarray(g, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty_like(g)
    err = ctypes.create_string_buffer(512)
    _check(lib().orc_training_mean(_p(g), _p(v), g.size, n, n_val, _p(out), err, 512), err)
    return out


def training_std(mean_t, sum_t, sum_sq_t, n_train):
    """fast.hpp:53-69."""
    a = [np.ascontiguousarray(t, np.float64) for t in (mean_t, sum_t, sum_sq_t)]
    out = np.empty_like(a[0])
    err = ctypes.create_string_buffer(512)
    _check(lib().orc_training_std(*[_p(t) for t in a], a[0].size, n_train, _p(out), err, 512), err)
    return out


@dataclass
class FoldResult:
    fold_id: int
    xtx_t: np.ndarray
    xty_t: np.ndarray
    mean_x_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    mean_y_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    std_x_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    std_y_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    n_train: int = 0
    n_val: int = 0


def _fold_result(fold_id, cfg, xtx, xty, mx, my, sx, sy, nt, nv):
    e = np.empty(0)
    return FoldResult(fold_id, xtx, xty, mx if cfg & 15 else e, my if cfg & 15 else e,
                      sx if cfg & SX else e, sy if cfg & SY else e, int(nt), int(nv))


def fold_products(cache: Cache, x, y, v_rows, cfg, fold_id=0) -> FoldResult:
    """fast.hpp:73-130 (single-fold entry point)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    n, k = x.shape
    m = y.shape[1]
    v = np.ascontiguousarray(v_rows, np.int64)
    xtx, xty = np.empty((k, k)), np.empty((k, m))
    mx, my, sx, sy = np.zeros(k), np.zeros(m), np.zeros(k), np.zeros(m)
    nt = np.zeros(1, np.int64)

    def vec(a, size):
        return a if a.size else np.zeros(size)

    cv = [vec(cache.sum_x, k), vec(cache.sum_y, m), vec(cache.mean_x, k), vec(cache.mean_y, m),
          vec(cache.sum_sq_x, k), vec(cache.sum_sq_y, m)]
    err = ctypes.create_string_buffer(512)
    _check(lib().orc_fold_products(_p(x), _p(y), cache.n_rows, k, m, _p(cache.xtx), _p(cache.xty),
                                   *[_p(a) for a in cv], _p(v), v.size, cfg, _p(xtx), _p(xty), _p(mx), _p(my),
                                   _p(sx), _p(sy), _p(nt), err, 512), err)
    return _fold_result(fold_id, cfg, xtx, xty, mx, my, sx, sy, nt[0], v.size)


def baseline_single_fold(x, y, v_rows, cfg, fold_id=0) -> FoldResult:
    """baseline.hpp:42-76."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    n, k = x.shape
    m = y.shape[1]
    v = np.ascontiguousarray(v_rows, np.int64)
    xtx, xty = np.empty((k, k)), np.empty((k, m))
    mx, my, sx, sy = np.zeros(k), np.zeros(m), np.zeros(k), np.zeros(m)
    nt = np.zeros(1, np.int64)
    err = ctypes.create_string_buffer(512)
    _check(lib().orc_baseline_single_fold(_p(x), _p(y), n, k, m, _p(v), v.size, cfg, _p(xtx), _p(xty), _p(mx),
                                          _p(my), _p(sx), _p(sy), _p(nt), err, 512), err)
    return _fold_result(fold_id, cfg, xtx, xty, mx, my, sx, sy, nt[0], v.size)


def _all_folds(fn, x, y, labels, p, cfg, n_threads, truth=False):
    labels = np.ascontiguousarray(labels, np.int32)
    if truth and np.asarray(x).dtype == np.float32:
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        f32 = 1
    else:
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        f32 = 0
    n, k = x.shape
    m = y.shape[1]
    pp = max(p, 0)
    xtx, xty = np.empty((pp, k, k)), np.empty((pp, k, m))
    mx, my, sx, sy = np.zeros((pp, k)), np.zeros((pp, m)), np.zeros((pp, k)), np.zeros((pp, m))
    nt, nv = np.zeros(pp, np.int64), np.zeros(pp, np.int64)
    err = ctypes.create_string_buffer(512)
    head = [_p(x), _p(y)] + ([f32] if truth else []) + [n, k, m, _p(labels), labels.size, p, cfg, n_threads]
    _check(fn(*head, _p(xtx), _p(xty), _p(mx), _p(my), _p(sx), _p(sy), _p(nt), _p(nv), err, 512), err)
    return [_fold_result(f + 1, cfg, xtx[f], xty[f], mx[f], my[f], sx[f], sy[f], nt[f], nv[f]) for f in range(p)]


def fast_all_folds(x, y, labels, p, cfg, n_threads=1):
    """R64: run_all_folds, fast.hpp:133-152."""
    return _all_folds(lib().orc_fast_all_folds, x, y, labels, p, cfg, n_threads)


def baseline_all_folds(x, y, labels, p, cfg, n_threads=1):
    """B64: baseline_fold_products, baseline.hpp:79-97."""
    return _all_folds(lib().orc_baseline_all_folds, x, y, labels, p, cfg, n_threads)


def truth_all_folds(x, y, labels, p, cfg, n_threads=1):
    """RLD: Algorithm 7 in long double in a globally shifted basis (the parity anchor)."""
    return _all_folds(lib().orc_truth_all_folds, x, y, labels, p, cfg, n_threads, truth=True)


def truth_all_folds_multi(x, y, labels, p, cfgs, n_threads=1):
    """RLD for several configurations from one long-double Gram pass: one list of folds per configuration."""
    labels = np.ascontiguousarray(labels, np.int32)
    f32 = 1 if np.asarray(x).dtype == np.float32 else 0
    dt = np.float32 if f32 else np.float64
    x = np.ascontiguousarray(x, dt)
    y = np.ascontiguousarray(y, dt)
    n, k = x.shape
    m = y.shape[1]
    nc = len(cfgs)
    cm = np.ascontiguousarray(cfgs, np.uint32)
    xtx, xty = np.empty((nc, p, k, k)), np.empty((nc, p, k, m))
    mx, my, sx, sy = np.zeros((nc, p, k)), np.zeros((nc, p, m)), np.zeros((nc, p, k)), np.zeros((nc, p, m))
    nt, nv = np.zeros(p, np.int64), np.zeros(p, np.int64)
    err = ctypes.create_string_buffer(512)
    _check(lib().orc_truth_all_folds_multi(_p(x), _p(y), f32, n, k, m, _p(labels), labels.size, p, _p(cm), nc,
                                           n_threads, _p(xtx), _p(xty), _p(mx), _p(my), _p(sx), _p(sy), _p(nt),
                                           _p(nv), err, 512), err)
    return [[_fold_result(f + 1, cfg, xtx[c, f], xty[c, f], mx[c, f], my[c, f], sx[c, f], sy[c, f], nt[f], nv[f])
             for f in range(p)] for c, cfg in enumerate(cfgs)]
