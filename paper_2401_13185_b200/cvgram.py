"""Python mirror of the reference `cvgram` API, backed by the B200 engine.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/cvgram/{core,partition,fast,random,combos}.hpp),
so the reference's Catch2 tests restate almost verbatim (tests/).  Every compute
call goes through the C ABI (include/cvgram_b200.h) into sm_100a kernels; the
host side here only validates, allocates and reshapes.

Exceptions mirror core.hpp:20-32: ``InvalidArgument`` stands for
std::invalid_argument and is the base of ``DimensionError``, ``PartitionError``
and ``ScalabilityError``.
"""
from __future__ import annotations

import ctypes
import os
import weakref
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


# ----------------------------------------------------------------- errors
class InvalidArgument(ValueError):
    """std::invalid_argument."""


class DimensionError(InvalidArgument):
    """cvgram::dimension_error (core.hpp:20-22)."""


class PartitionError(InvalidArgument):
    """cvgram::partition_error (core.hpp:24-26)."""


class ScalabilityError(InvalidArgument):
    """cvgram::scalability_error (core.hpp:30-32)."""


class DeviceError(RuntimeError):
    """The B200 engine could not run (no device, CUDA failure, out of memory)."""


_ERRORS = {L.E_DIMENSION: DimensionError, L.E_PARTITION: PartitionError, L.E_SCALABILITY: ScalabilityError,
           L.E_INVALID_ARG: InvalidArgument, L.E_CUDA: DeviceError, L.E_OOM: DeviceError, L.E_NCCL: DeviceError}


def _check(rc: int, buf) -> None:
    if rc != L.OK:
        raise _ERRORS.get(rc, DeviceError)(buf.value.decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------- context
class Context:
    """A device binding (cvg_context): stream, launch counter, reusable scratch."""

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        buf = L.err_buf()
        _check(L.lib().cvg_context_create(device, ctypes.byref(h), buf, len(buf)), buf)
        self._h = h
        self._fin = weakref.finalize(self, L.lib().cvg_context_destroy, h)

    @property
    def handle(self):
        return self._h

    @property
    def launches(self) -> int:
        return int(L.lib().cvg_context_launch_count(self._h))

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """cudaStream_t handle; None = the context's own stream.  A torch stream
        handle of 0 is the legacy default stream: pass it as cudaStreamLegacy (1),
        since NULL would select the context's own (non-blocking) stream."""
        L.lib().cvg_context_set_stream(self._h, stream_ptr)

    def use_torch_stream(self, stream) -> None:
        """Issue subsequent work on a torch.cuda.Stream (ordered after torch's copies)."""
        self.set_stream(stream.cuda_stream or CUDA_STREAM_LEGACY)

    def close(self) -> None:
        self._fin()


class MultiContext(Context):
    """Several devices behind one context (cvg_context_create_multi): run_all_folds on it shards the folds
    across the devices (per-device host threads; NCCL exchanges over distinct devices, device copies when a
    device repeats -- a one-GPU emulation), bit-identical to one device.  Other calls run on devices[0]."""

    def __init__(self, devices):
        self.devices = [int(d) for d in devices]
        self.device = self.devices[0]
        ids = (ctypes.c_int * len(self.devices))(*self.devices)
        h = ctypes.c_void_p()
        buf = L.err_buf()
        _check(L.lib().cvg_context_create_multi(len(self.devices), ids, ctypes.byref(h), buf, len(buf)), buf)
        self._h = h
        self._fin = weakref.finalize(self, L.lib().cvg_context_destroy, h)

    @property
    def device_count(self) -> int:
        return int(L.lib().cvg_context_device_count(self._h))

    @property
    def exchange(self) -> str:
        return {1: "nccl", 2: "copy"}.get(int(L.lib().cvg_context_exchange(self._h)), "single")


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy
_contexts: dict = {}


def default_device() -> int:
    return int(os.environ.get("CVG_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def get_context(device: Optional[int] = None) -> Context:
    d = default_device() if device is None else device
    if d not in _contexts:
        _contexts[d] = Context(d)
    return _contexts[d]


# ------------------------------------------------------------- core types
@dataclass(frozen=True)
class PreprocessConfig:
    """Four independent flags (core.hpp:67-78)."""

    center_x: bool = False
    center_y: bool = False
    scale_x: bool = False
    scale_y: bool = False

    def any_center(self) -> bool:
        return self.center_x or self.center_y

    def any_scale(self) -> bool:
        return self.scale_x or self.scale_y

    def any(self) -> bool:
        return self.any_center() or self.any_scale()

    @property
    def mask(self) -> int:
        """enumerate_configs bit order (combos.hpp:33-45)."""
        return (8 if self.center_x else 0) | (4 if self.center_y else 0) | (2 if self.scale_x else 0) | (
            1 if self.scale_y else 0)

    @staticmethod
    def from_mask(bits: int) -> "PreprocessConfig":
        return PreprocessConfig(bool(bits & 8), bool(bits & 4), bool(bits & 2), bool(bits & 1))


def enumerate_configs() -> List[PreprocessConfig]:
    """All 16 flag combinations as a 4-bit counter, all-off first (combos.hpp:33-45)."""
    return [PreprocessConfig.from_mask(b) for b in range(16)]


def _cfg(cfg) -> PreprocessConfig:
    if cfg is None:
        return PreprocessConfig()
    if isinstance(cfg, PreprocessConfig):
        return cfg
    if isinstance(cfg, int):
        return PreprocessConfig.from_mask(cfg)
    return PreprocessConfig(*cfg)


class DatasetPair:
    """X (N x K) and Y (N x M), one sample per row (core.hpp:35-56).

    fp64 is the reference type; fp32 inputs are accepted for the fp32 path
    (BASELINE.json configs[3]).  Validation is core.hpp:38-44, in order.
    """

    def __init__(self, x, y):
        x = np.asarray(x)
        y = np.asarray(y)
        dt = np.float32 if (x.dtype == np.float32 and y.dtype == np.float32) else np.float64
        x = np.ascontiguousarray(x, dt)
        y = np.ascontiguousarray(y, dt)
        if x.ndim != 2 or y.ndim != 2:
            raise DimensionError("x and y must be matrices")
        if x.shape[0] != y.shape[0]:
            raise DimensionError("x and y must have the same number of rows")
        if x.shape[0] < 2:
            raise DimensionError("need at least 2 samples")
        if x.shape[1] < 1 or y.shape[1] < 1:
            raise DimensionError("x and y must each have at least one column")
        if not (np.isfinite(x).all() and np.isfinite(y).all()):
            raise DimensionError("x and y entries must be finite")
        x.setflags(write=False)
        y.setflags(write=False)
        self._x, self._y = x, y

    def x(self) -> np.ndarray:
        return self._x

    def y(self) -> np.ndarray:
        return self._y

    def n_rows(self) -> int:
        return self._x.shape[0]

    def n_features(self) -> int:
        return self._x.shape[1]

    def n_responses(self) -> int:
        return self._y.shape[1]

    @property
    def dtype_code(self) -> int:
        return L.DTYPE_F32 if self._x.dtype == np.float32 else L.DTYPE_F64


@dataclass
class Partitioning:
    """Length-N 1-based fold labels and the fold count p (core.hpp:59-64)."""

    labels: np.ndarray
    p: int = 0

    def __post_init__(self):
        self.labels = np.ascontiguousarray(self.labels, np.int32)

    def n_rows(self) -> int:
        return int(self.labels.size)


def _empty():
    return np.empty(0)


_EMPTY = np.empty(0)
_EMPTY.flags.writeable = False  # the shared "not filled" statistic (FoldStats fill rules, core.hpp:95-105)
_PINNED_MIN_BYTES = 1 << 22


def _output_array(shape, dtype=np.float64):
    """An output array for the engine's device-to-host copies: large ones come from the library's pinned host
    pool (cvg_host_alloc; the block returns to the pool when the array -- and every view of it -- is gone), so
    results land at full PCIe speed in already-faulted pages; small ones, or no pool, are plain np.empty."""
    shape = tuple(int(d) for d in shape)
    nbytes = int(np.prod(shape, dtype=np.int64)) * np.dtype(dtype).itemsize
    if nbytes < _PINNED_MIN_BYTES:
        return np.empty(shape, dtype)
    p = ctypes.c_void_p()
    if L.lib().cvg_host_alloc(nbytes, ctypes.byref(p)) != L.OK or not p.value:
        return np.empty(shape, dtype)
    raw = (ctypes.c_char * nbytes).from_address(p.value)
    arr = np.frombuffer(raw, dtype=dtype).reshape(shape)
    weakref.finalize(raw, L.lib().cvg_host_free, ctypes.c_void_p(p.value))
    return arr


@dataclass
class GlobalCache:
    """Whole-dataset aggregates (core.hpp:83-93); unused vectors stay empty."""

    xtx: np.ndarray
    xty: np.ndarray
    mean_x: np.ndarray = field(default_factory=_empty)
    mean_y: np.ndarray = field(default_factory=_empty)
    sum_x: np.ndarray = field(default_factory=_empty)
    sum_y: np.ndarray = field(default_factory=_empty)
    sum_sq_x: np.ndarray = field(default_factory=_empty)
    sum_sq_y: np.ndarray = field(default_factory=_empty)
    n_rows: int = 0
    _device: object = field(default=None, repr=False, compare=False)


@dataclass
class FoldStats:
    """Training statistics actually used for one fold (core.hpp:98-105)."""

    mean_x_t: np.ndarray = field(default_factory=_empty)
    mean_y_t: np.ndarray = field(default_factory=_empty)
    std_x_t: np.ndarray = field(default_factory=_empty)
    std_y_t: np.ndarray = field(default_factory=_empty)
    n_train: int = 0
    n_val: int = 0


@dataclass
class FoldResult:
    """core.hpp:107-112."""

    fold_id: int
    xtx_t: np.ndarray
    xty_t: np.ndarray
    stats: FoldStats = field(default_factory=FoldStats)


# ------------------------------------------------------------- partition.hpp
@dataclass
class ValidationIndex:
    sets: List[np.ndarray]


def _labels_p(part_or_labels, p=None):
    if isinstance(part_or_labels, Partitioning):
        return part_or_labels.labels, part_or_labels.p
    return np.ascontiguousarray(part_or_labels, np.int32), int(p)


def validate_partitioning(part_or_labels, p: Optional[int] = None) -> Optional[str]:
    """None if valid, else the first violated clause (partition.hpp:21-45)."""
    labels, p = _labels_p(part_or_labels, p)
    buf = L.err_buf()
    rc = L.lib().cvg_validate_partitioning(_ptr(labels), labels.size, p, buf, len(buf))
    return None if rc == L.OK else buf.value.decode()


def check_scalable(part: Partitioning) -> Optional[str]:
    """None iff every training partition has >= 2 rows (partition.hpp:48-58)."""
    buf = L.err_buf()
    rc = L.lib().cvg_check_scalable(_ptr(part.labels), part.labels.size, part.p, buf, len(buf))
    return None if rc == L.OK else buf.value.decode()


def build_validation_partitions(part: Partitioning) -> ValidationIndex:
    """Ascending 0-based row lists per fold (partition.hpp:61-68).  Index
    bookkeeping only; the engine buckets rows on the device itself."""
    order = np.argsort(part.labels, kind="stable")
    counts = np.bincount(part.labels - 1, minlength=part.p)[: part.p]
    bounds = np.concatenate([[0], np.cumsum(counts)])
    return ValidationIndex([order[bounds[f]:bounds[f + 1]].astype(np.int64) for f in range(part.p)])


def complement_rows(v_rows, n: int) -> np.ndarray:
    """Rows not in v_rows, ascending (partition.hpp:71-83)."""
    mask = np.ones(n, bool)
    mask[np.asarray(v_rows, np.int64)] = False
    return np.nonzero(mask)[0].astype(np.int64)


def gather_rows(src: np.ndarray, rows) -> np.ndarray:
    """partition.hpp:85-90."""
    return np.ascontiguousarray(src[np.asarray(rows, np.int64)])


# ------------------------------------------------------------------ core.hpp
def hadamard_outer_divide(mat, left, right, ctx: Optional[Context] = None) -> np.ndarray:
    """out(i,j) = m(i,j) / (left(i) * right(j)) on the device (core.hpp:116-130)."""
    ctx = ctx or get_context()
    mat = np.ascontiguousarray(np.atleast_2d(mat), np.float64)
    left = np.ascontiguousarray(left, np.float64).ravel()
    right = np.ascontiguousarray(right, np.float64).ravel()
    out = np.empty_like(mat)
    buf = L.err_buf()
    _check(L.lib().cvg_hadamard_outer_divide(ctx.handle, _ptr(mat), mat.shape[0], mat.shape[1], _ptr(left),
                                             left.size, _ptr(right), right.size, _ptr(out), buf, len(buf)), buf)
    return out


def max_rel_diff(a, b, floor: float = 1e-30) -> float:
    """Largest entrywise |a-b| / max(|a|, |b|, floor) (core.hpp:133-150)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise DimensionError("max_rel_diff: shape mismatch")
    if a.size == 0:
        return 0.0
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / den))


def rel_frobenius_dist(a, b, floor: float = 1e-30) -> float:
    """||a-b||_F / max(||a||_F, ||b||_F, floor) (core.hpp:153-156)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), np.linalg.norm(b), floor))


# ------------------------------------------------------------------ fast.hpp
class _DeviceGlobal:
    """Owns a cvg_global: the shifted-basis whole-data Gram kept on the device."""

    def __init__(self, ctx: Context, data: DatasetPair):
        self.ctx = ctx
        self.data = data
        h = ctypes.c_void_p()
        buf = L.err_buf()
        _check(L.lib().cvg_global_create(ctx.handle, data.dtype_code, _ptr(data.x()), _ptr(data.y()), data.n_rows(),
                                         data.n_features(), data.n_responses(), ctypes.byref(h), buf, len(buf)), buf)
        self.h = h
        self._fin = weakref.finalize(self, L.lib().cvg_global_destroy, h)


def precompute_global(data: DatasetPair, cfg=None, ctx: Optional[Context] = None) -> GlobalCache:
    """Whole-dataset products and the statistic vectors cfg needs (fast.hpp:19-36)."""
    cfg = _cfg(cfg)
    ctx = ctx or get_context()
    dev = _DeviceGlobal(ctx, data)
    k, m = data.n_features(), data.n_responses()
    xtx, xty = np.empty((k, k)), np.empty((k, m))
    vec = {name: np.empty(k if name.endswith("x") else m) for name in
           ("sum_x", "sum_y", "mean_x", "mean_y", "sum_sq_x", "sum_sq_y")}
    buf = L.err_buf()
    _check(L.lib().cvg_global_export(dev.h, cfg.mask, _ptr(xtx), _ptr(xty), *[_ptr(vec[n]) for n in (
        "sum_x", "sum_y", "mean_x", "mean_y", "sum_sq_x", "sum_sq_y")], buf, len(buf)), buf)
    cache = GlobalCache(xtx, xty, n_rows=data.n_rows(), _device=dev)
    if cfg.any():
        cache.sum_x, cache.sum_y, cache.mean_x, cache.mean_y = vec["sum_x"], vec["sum_y"], vec["mean_x"], vec["mean_y"]
    if cfg.any_scale():
        cache.sum_sq_x, cache.sum_sq_y = vec["sum_sq_x"], vec["sum_sq_y"]
    return cache


def training_mean(global_mean, val_mean, n: int, n_val: int, ctx: Optional[Context] = None) -> np.ndarray:
    """(n/(n-n_val))·global − (n_val/(n-n_val))·val, on the device (fast.hpp:40-47)."""
    ctx = ctx or get_context()
    g = np.ascontiguousarray(global_mean, np.float64).ravel()
    v = np.ascontiguousarray(val_mean, np.float64).ravel()
    out = np.empty_like(g)
    buf = L.err_buf()
    _check(L.lib().cvg_training_mean(ctx.handle, _ptr(g), _ptr(v), g.size, n, n_val, _ptr(out), buf, len(buf)), buf)
    return out


def training_std(mean_t, sum_t, sum_sq_t, n_train: int, ctx: Optional[Context] = None) -> np.ndarray:
    """Bessel-corrected std from training sums, clamp and zero->1 (fast.hpp:53-69)."""
    ctx = ctx or get_context()
    a = [np.ascontiguousarray(t, np.float64).ravel() for t in (mean_t, sum_t, sum_sq_t)]
    out = np.empty_like(a[0])
    buf = L.err_buf()
    _check(L.lib().cvg_training_std(ctx.handle, *[_ptr(t) for t in a], a[0].size, n_train, _ptr(out), buf,
                                    len(buf)), buf)
    return out


def fold_products(cache: GlobalCache, data: DatasetPair, v_rows: Sequence[int], cfg=None, fold_id: int = 0,
                  ctx: Optional[Context] = None) -> FoldResult:
    """Training products for one fold from the cache + validation rows (fast.hpp:73-130)."""
    cfg = _cfg(cfg)
    dev = cache._device
    if dev is None or dev.data is not data:
        dev = _DeviceGlobal(ctx or get_context(), data)
        cache._device = dev
    k, m = data.n_features(), data.n_responses()
    v = np.ascontiguousarray(v_rows, np.int64)
    xtx, xty = np.empty((k, k)), np.empty((k, m))
    mx, my, sx, sy = np.empty(k), np.empty(m), np.empty(k), np.empty(m)
    nt = ctypes.c_int64(0)
    buf = L.err_buf()
    _check(L.lib().cvg_global_fold_products(dev.h, _ptr(v), v.size, cfg.mask, _ptr(xtx), _ptr(xty), _ptr(mx),
                                            _ptr(my), _ptr(sx), _ptr(sy), ctypes.addressof(nt), buf, len(buf)), buf)
    stats = FoldStats(n_train=int(nt.value), n_val=int(v.size))
    if cfg.any():
        stats.mean_x_t, stats.mean_y_t = mx, my
    if cfg.scale_x:
        stats.std_x_t = sx
    if cfg.scale_y:
        stats.std_y_t = sy
    return FoldResult(fold_id, xtx, xty, stats)


def run_all_folds_configs(data: DatasetPair, part: Partitioning, cfgs, ctx: Optional[Context] = None):
    """run_all_folds for several configurations with one Gram pass.

    Returns one list of FoldResult (ascending fold_id) per configuration.
    """
    cfgs = [_cfg(c) for c in cfgs]
    ctx = ctx or get_context()
    n, k, m, p = data.n_rows(), data.n_features(), data.n_responses(), part.p
    nc = len(cfgs)
    pp = max(p, 0)
    masks = np.array([c.mask for c in cfgs], np.uint32)
    xtx = _output_array((nc, pp, k, k))
    xty = _output_array((nc, pp, k, m))
    mx, my = _output_array((nc, pp, k)), _output_array((nc, pp, m))
    sx, sy = _output_array((nc, pp, k)), _output_array((nc, pp, m))
    nt, nv = np.empty(pp, np.int64), np.empty(pp, np.int64)
    buf = L.err_buf()
    _check(L.lib().cvg_run_all_folds(ctx.handle, data.dtype_code, _ptr(data.x()), _ptr(data.y()), n, k, m,
                                     _ptr(part.labels), part.labels.size, p, _ptr(masks), nc, _ptr(xtx), _ptr(xty),
                                     _ptr(mx), _ptr(my), _ptr(sx), _ptr(sy), _ptr(nt), _ptr(nv), buf, len(buf)), buf)
    out = []
    ntl, nvl = nt.tolist(), nv.tolist()
    for ci, cfg in enumerate(cfgs):
        anyc, scx, scy = cfg.any(), cfg.scale_x, cfg.scale_y
        xs, ys, mxs, mys, sxs, sys_ = xtx[ci], xty[ci], mx[ci], my[ci], sx[ci], sy[ci]
        runs = []
        for f in range(p):
            st = FoldStats(mxs[f] if anyc else _EMPTY, mys[f] if anyc else _EMPTY, sxs[f] if scx else _EMPTY,
                           sys_[f] if scy else _EMPTY, ntl[f], nvl[f])
            runs.append(FoldResult(f + 1, xs[f], ys[f], st))
        out.append(runs)
    return out


_FOLD_BATCH_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int32, ctypes.c_int32, *([ctypes.c_void_p] * 9))


def for_each_fold(data: DatasetPair, part: Partitioning, cfgs, fn, batch: int = 1024,
                  ctx: Optional[Context] = None) -> None:
    """Lazy per-fold generation (cvg_run_all_folds_stream): ``fn(config_index, FoldResult)`` is called for every
    configuration and fold, folds in ascending order, while only ``batch`` folds of outputs exist at a time
    (leave-one-out-scale P).  ``fn`` returning True stops the run.  Same values as run_all_folds_configs."""
    cfgs = [_cfg(c) for c in cfgs]
    ctx = ctx or get_context()
    n, k, m, p = data.n_rows(), data.n_features(), data.n_responses(), part.p
    nc = len(cfgs)
    masks = np.array([c.mask for c in cfgs], np.uint32)
    stop = [False]
    error = []

    def on_batch(lo, hi, pxx, pxy, pmx, pmy, psx, psy, pnt, pnv, _user):
        try:
            nb = hi - lo
            arr = lambda ptr, shape, dt=np.float64: np.ctypeslib.as_array(  # noqa: E731
                ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double if dt == np.float64 else ctypes.c_int64)), shape)
            xtx, xty = arr(pxx, (nc, nb, k, k)), arr(pxy, (nc, nb, k, m))
            mx, my, sx, sy = arr(pmx, (nb, k)), arr(pmy, (nb, m)), arr(psx, (nb, k)), arr(psy, (nb, m))
            nt, nv = arr(pnt, (nb,), np.int64), arr(pnv, (nb,), np.int64)
            for f in range(nb):
                for ci, cfg in enumerate(cfgs):
                    st = FoldStats(n_train=int(nt[f]), n_val=int(nv[f]))
                    if cfg.any():
                        st.mean_x_t, st.mean_y_t = mx[f].copy(), my[f].copy()
                    if cfg.scale_x:
                        st.std_x_t = sx[f].copy()
                    if cfg.scale_y:
                        st.std_y_t = sy[f].copy()
                    if fn(ci, FoldResult(lo + f + 1, xtx[ci, f].copy(), xty[ci, f].copy(), st)):
                        stop[0] = True
                        return 1
            return 0
        except BaseException as e:  # surface Python errors after the C call returns
            error.append(e)
            return 1

    cb = _FOLD_BATCH_FN(on_batch)
    buf = L.err_buf()
    _check(L.lib().cvg_run_all_folds_stream(ctx.handle, data.dtype_code, _ptr(data.x()), _ptr(data.y()), n, k, m,
                                            _ptr(part.labels), part.labels.size, p, _ptr(masks), nc, int(batch),
                                            ctypes.cast(cb, ctypes.c_void_p), None, buf, len(buf)), buf)
    if error:
        raise error[0]


def run_all_folds(data: DatasetPair, part: Partitioning, cfg=None, n_threads: int = 1,
                  ctx: Optional[Context] = None) -> List[FoldResult]:
    """One global pass, then every fold; ascending fold_id (fast.hpp:133-152).

    n_threads is accepted for signature parity; the device grid replaces the
    fold thread pool and results never depend on it (threading.hpp:8-10).
    """
    if part.n_rows() != data.n_rows():
        raise DimensionError("partitioning length does not match sample count")
    return run_all_folds_configs(data, part, [_cfg(cfg)], ctx)[0]


# ---------------------------------------------------------------- random.hpp
class MT19937_64:
    """std::mt19937_64 stream (random.hpp:14-18) via the engine library."""

    def __init__(self, seed: int):
        self._h = L.lib().cvg_rng_create(seed)
        self._fin = weakref.finalize(self, L.lib().cvg_rng_destroy, self._h)

    def __call__(self) -> int:
        return int(L.lib().cvg_rng_next(self._h))

    def uniform01(self) -> float:
        return float(L.lib().cvg_rng_uniform01(self._h))

    @property
    def handle(self):
        return self._h


def _rng(rng_or_seed) -> MT19937_64:
    return rng_or_seed if isinstance(rng_or_seed, MT19937_64) else MT19937_64(int(rng_or_seed))


def uniform01(rng: MT19937_64) -> float:
    return rng.uniform01()


def random_dataset(n: int, k: int, m: int, rng) -> DatasetPair:
    """Row-major fill, X first then Y, from one stream (random.hpp:21-33)."""
    rng = _rng(rng)
    x, y = np.empty((n, k)), np.empty((n, m))
    L.lib().cvg_random_dataset(rng.handle, n, k, m, _ptr(x), _ptr(y))
    return DatasetPair(x, y)


def random_partitioning(n: int, p: int, rng) -> Partitioning:
    """Balanced labels 1 + (i mod p), then Fisher-Yates (random.hpp:38-55)."""
    rng = _rng(rng)
    labels = np.empty(n, np.int32)
    L.lib().cvg_random_partitioning(rng.handle, n, p, _ptr(labels))
    return Partitioning(labels, p)


# ---------------------------------------------------------------- baseline.hpp
def baseline_fold_products_configs(data: DatasetPair, part: Partitioning, cfgs, ctx: Optional[Context] = None):
    """The baseline engine (baseline.hpp:79-97) on the device for several
    configurations: per fold, the training rows are contracted directly in
    their own mean-centered basis — no downdate.  Θ(P·N·K(K+M))."""
    cfgs = [_cfg(c) for c in cfgs]
    ctx = ctx or get_context()
    if part.n_rows() != data.n_rows():
        raise DimensionError("partitioning length does not match sample count")
    n, k, m, p = data.n_rows(), data.n_features(), data.n_responses(), part.p
    nc, pp = len(cfgs), max(p, 0)
    masks = np.array([c.mask for c in cfgs], np.uint32)
    xtx, xty = np.empty((nc, pp, k, k)), np.empty((nc, pp, k, m))
    mx, my, sx, sy = np.empty((nc, pp, k)), np.empty((nc, pp, m)), np.empty((nc, pp, k)), np.empty((nc, pp, m))
    nt, nv = np.empty(pp, np.int64), np.empty(pp, np.int64)
    buf = L.err_buf()
    _check(L.lib().cvg_baseline_fold_products(ctx.handle, data.dtype_code, _ptr(data.x()), _ptr(data.y()), n, k, m,
                                              _ptr(part.labels), part.labels.size, p, _ptr(masks), nc, _ptr(xtx),
                                              _ptr(xty), _ptr(mx), _ptr(my), _ptr(sx), _ptr(sy), _ptr(nt), _ptr(nv),
                                              buf, len(buf)), buf)
    out = []
    ntl, nvl = nt.tolist(), nv.tolist()
    for ci, cfg in enumerate(cfgs):
        anyc, scx, scy = cfg.any(), cfg.scale_x, cfg.scale_y
        xs, ys, mxs, mys, sxs, sys_ = xtx[ci], xty[ci], mx[ci], my[ci], sx[ci], sy[ci]
        runs = []
        for f in range(p):
            st = FoldStats(mxs[f] if anyc else _EMPTY, mys[f] if anyc else _EMPTY, sxs[f] if scx else _EMPTY,
                           sys_[f] if scy else _EMPTY, ntl[f], nvl[f])
            runs.append(FoldResult(f + 1, xs[f], ys[f], st))
        out.append(runs)
    return out


def baseline_fold_products(data: DatasetPair, part: Partitioning, cfg=None, n_threads: int = 1,
                           ctx: Optional[Context] = None) -> List[FoldResult]:
    """baseline.hpp:79-97 (n_threads accepted for signature parity)."""
    return baseline_fold_products_configs(data, part, [_cfg(cfg)], ctx)[0]


def baseline_single_fold(data: DatasetPair, v_rows: Sequence[int], cfg=None, fold_id: int = 0,
                         ctx: Optional[Context] = None) -> FoldResult:
    """baseline.hpp:42-76."""
    cfg = _cfg(cfg)
    ctx = ctx or get_context()
    k, m = data.n_features(), data.n_responses()
    v = np.ascontiguousarray(v_rows, np.int64)
    xtx, xty = np.empty((k, k)), np.empty((k, m))
    mx, my, sx, sy = np.empty(k), np.empty(m), np.empty(k), np.empty(m)
    nt = ctypes.c_int64(0)
    buf = L.err_buf()
    _check(L.lib().cvg_baseline_single_fold(ctx.handle, data.dtype_code, _ptr(data.x()), _ptr(data.y()),
                                            data.n_rows(), k, m, _ptr(v), v.size, cfg.mask, _ptr(xtx), _ptr(xty),
                                            _ptr(mx), _ptr(my), _ptr(sx), _ptr(sy), ctypes.addressof(nt), buf,
                                            len(buf)), buf)
    stats = FoldStats(n_train=int(nt.value), n_val=int(v.size))
    if cfg.any():
        stats.mean_x_t, stats.mean_y_t = mx, my
    if cfg.scale_x:
        stats.std_x_t = sx
    if cfg.scale_y:
        stats.std_y_t = sy
    return FoldResult(fold_id, xtx, xty, stats)


# ------------------------------------------------------------------ combos.hpp
@dataclass
class ComboClassReport:
    """combos.hpp:21-31."""

    configs: List[PreprocessConfig]
    xty_class: List[int]
    pair_class: List[int]
    n_xty_classes: int
    n_pair_classes: int
    min_xty_separation: float
    min_pair_separation: float
    tol: float
    degenerate: bool


def _group_classes(runs, tol, dist):
    """combos.hpp:69-94: first-fit grouping in canonical order."""
    reps, cls, min_sep = [], [], float("inf")
    for c in range(16):
        assigned = -1
        for kidx, rep in enumerate(reps):
            d = dist(runs[c], runs[rep])
            if d <= tol and assigned < 0:
                assigned = kidx
            elif d > tol:
                min_sep = min(min_sep, d)
        if assigned < 0:
            assigned = len(reps)
            reps.append(c)
        cls.append(assigned)
    if len(reps) <= 1:
        min_sep = 0.0
    return len(reps), cls, min_sep


def classify_combos(data: DatasetPair, part: Partitioning, tol: float = 1e-9,
                    ctx: Optional[Context] = None) -> ComboClassReport:
    """Certify the 8 XᵀY / 12 (XᵀX, XᵀY) configuration classes (combos.hpp:98-120)
    over the engine's outputs; all 16 configurations come from one Gram pass."""
    err = check_scalable(part)
    if err:
        raise ScalabilityError(err)
    configs = enumerate_configs()
    runs = run_all_folds_configs(data, part, configs, ctx)

    def d_xty(a, b):
        return max(rel_frobenius_dist(x.xty_t, y.xty_t) for x, y in zip(a, b))

    def d_pair(a, b):
        return max(d_xty(a, b), max(rel_frobenius_dist(x.xtx_t, y.xtx_t) for x, y in zip(a, b)))

    nx, cx, sx = _group_classes(runs, tol, d_xty)
    np_, cp, sp = _group_classes(runs, tol, d_pair)
    return ComboClassReport(configs, cx, cp, nx, np_, sx, sp, tol, nx != 8 or np_ != 12)


def format_combo_table(report: ComboClassReport) -> str:
    """combos.hpp:124-161 (same text layout)."""
    centers = ["no centering", "center X", "center Y", "center both"]
    scales = ["no scaling", "scale X", "scale Y", "scale both"]

    def idx(ci, si):
        cx = 1 if ci in (1, 3) else 0
        cy = 1 if ci in (2, 3) else 0
        sx = 1 if si in (1, 3) else 0
        sy = 1 if si in (2, 3) else 0
        return (cx << 3) | (cy << 2) | (sx << 1) | sy

    lines = []

    def grid(title, cls):
        lines.append(title)
        lines.append("centering \\ scaling" + "".join("\t" + s for s in scales))
        for ci in range(4):
            lines.append(centers[ci] + "".join("\t" + str(cls[idx(ci, si)]) for si in range(4)))

    grid("XtY classes", report.xty_class)
    lines.append("")
    grid("(XtX, XtY) pair classes", report.pair_class)
    g = lambda v: "%g" % v  # noqa: E731  (std::ostream default formatting)
    text = "\n".join(lines) + "\n"
    text += (f"\ndistinct XtY classes: {report.n_xty_classes}\ndistinct pair classes: {report.n_pair_classes}"
             f"\nmin inter-class separation (xty): {g(report.min_xty_separation)}"
             f"\nmin inter-class separation (pair): {g(report.min_pair_separation)}\ntolerance: {g(report.tol)}\n")
    if report.degenerate:
        text += "warning: class counts are degenerate for this input; expected 8 xty and 12 pair classes\n"
    return text


# ---------------------------------------------------------------------- io.hpp
def format_double(v: float) -> str:
    """%.17g, the reference's round-trip format (io.hpp:24-28)."""
    return "%.17g" % v


def config_to_string(cfg) -> str:
    """4-bit token cx cy sx sy (io.hpp:115-122)."""
    c = _cfg(cfg)
    return "".join("1" if b else "0" for b in (c.center_x, c.center_y, c.scale_x, c.scale_y))


def parse_config(s: str) -> PreprocessConfig:
    """io.hpp:126-149."""
    if s == "none":
        return PreprocessConfig()
    if s == "center":
        return PreprocessConfig(True, True, False, False)
    if s == "scale":
        return PreprocessConfig(False, False, True, True)
    if s in ("center+scale", "center_scale"):
        return PreprocessConfig(True, True, True, True)
    if len(s) == 4 and set(s) <= {"0", "1"}:
        return PreprocessConfig(*(ch == "1" for ch in s))
    raise IOError(f"unknown preprocessing config '{s}'")
