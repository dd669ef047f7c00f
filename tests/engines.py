"""Adapters giving the oracle and the B200 engine one reference-shaped API, so
the reference's own test cases (tests/golden/reference_kats.json and the
restated Catch2 cases) run unchanged against both."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2401_13185_b200 import cvgram as cv

ERR_BY_CODE = {1: cv.DimensionError, 2: cv.PartitionError, 3: cv.ScalabilityError, 4: cv.InvalidArgument}
ERR_BY_NAME = {"invalid_argument": cv.InvalidArgument, "dimension_error": cv.DimensionError,
               "partition_error": cv.PartitionError, "scalability_error": cv.ScalabilityError}


@dataclass
class R:
    fold_id: int
    xtx_t: np.ndarray
    xty_t: np.ndarray
    mean_x_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    mean_y_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    std_x_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    std_y_t: np.ndarray = field(default_factory=lambda: np.empty(0))
    n_train: int = 0
    n_val: int = 0


def _flat(r) -> R:
    if hasattr(r, "stats"):
        s = r.stats
        return R(r.fold_id, r.xtx_t, r.xty_t, s.mean_x_t, s.mean_y_t, s.std_x_t, s.std_y_t, s.n_train, s.n_val)
    return R(r.fold_id, r.xtx_t, r.xty_t, r.mean_x_t, r.mean_y_t, r.std_x_t, r.std_y_t, r.n_train, r.n_val)


class OracleEngine:
    name = "oracle"

    def __init__(self):
        import oracle

        self.o = oracle

    def _call(self, fn, *a, **kw):
        try:
            return fn(*a, **kw)
        except self.o.OracleError as e:
            raise ERR_BY_CODE.get(e.code, cv.InvalidArgument)(str(e)) from e

    def precompute_global(self, x, y, cfg):
        return self._call(self.o.precompute_global, x, y, cfg)

    def fold_products(self, cache, x, y, v_rows, cfg, fold_id=0):
        return _flat(self._call(self.o.fold_products, cache, x, y, v_rows, cfg, fold_id))

    def run_all_folds(self, x, y, labels, p, cfg, n_threads=1):
        return [_flat(r) for r in self._call(self.o.fast_all_folds, x, y, labels, p, cfg, n_threads)]

    def run_all_folds_configs(self, x, y, labels, p, cfgs):
        return [self.run_all_folds(x, y, labels, p, c) for c in cfgs]

    def baseline_all_folds(self, x, y, labels, p, cfg):
        return [_flat(r) for r in self._call(self.o.baseline_all_folds, x, y, labels, p, cfg)]

    def baseline_single_fold(self, x, y, v_rows, cfg, fold_id=0):
        return _flat(self._call(self.o.baseline_single_fold, x, y, v_rows, cfg, fold_id))

    def training_mean(self, g, v, n, n_val):
        return self._call(self.o.training_mean, g, v, n, n_val)

    def training_std(self, m, s, q, n_train):
        return self._call(self.o.training_std, m, s, q, n_train)

    def hadamard_outer_divide(self, m, l, r):
        return self._call(self.o.hadamard_outer_divide, m, l, r)


class GpuEngine:
    name = "gpu"

    def precompute_global(self, x, y, cfg):
        return cv.precompute_global(cv.DatasetPair(x, y), cfg)

    def fold_products(self, cache, x, y, v_rows, cfg, fold_id=0):
        data = cache._device.data if cache._device is not None else cv.DatasetPair(x, y)
        return _flat(cv.fold_products(cache, data, v_rows, cfg, fold_id))

    def run_all_folds(self, x, y, labels, p, cfg, n_threads=1):
        return [_flat(r) for r in cv.run_all_folds(cv.DatasetPair(x, y), cv.Partitioning(labels, p), cfg, n_threads)]

    def run_all_folds_configs(self, x, y, labels, p, cfgs):
        runs = cv.run_all_folds_configs(cv.DatasetPair(x, y), cv.Partitioning(labels, p), cfgs)
        return [[_flat(r) for r in run] for run in runs]

    def baseline_all_folds(self, x, y, labels, p, cfg):
        return [_flat(r) for r in cv.baseline_fold_products(cv.DatasetPair(x, y), cv.Partitioning(labels, p), cfg)]

    def baseline_single_fold(self, x, y, v_rows, cfg, fold_id=0):
        return _flat(cv.baseline_single_fold(cv.DatasetPair(x, y), v_rows, cfg, fold_id))

    def training_mean(self, g, v, n, n_val):
        return cv.training_mean(g, v, n, n_val)

    def training_std(self, m, s, q, n_train):
        return cv.training_std(m, s, q, n_train)

    def hadamard_outer_divide(self, m, l, r):
        return cv.hadamard_outer_divide(m, l, r)


def make(name):
    return OracleEngine() if name == "oracle" else GpuEngine()


def normalized_err(got, ref, diag_ref_i=None, diag_ref_j=None):
    """|Δ_ij| / max(|ref_ij|, sqrt(|D_i D_j|)) — the floored entrywise metric of
    SURVEY.md §8(d); D are the diagonal second moments of the two sides."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    if diag_ref_i is None:
        d = np.sqrt(np.abs(np.diag(ref)))
        scale = np.outer(d, d)
    else:
        scale = np.sqrt(np.outer(np.abs(diag_ref_i), np.abs(diag_ref_j)))
    den = np.maximum(np.abs(ref), scale)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(np.abs(got - ref) / den)) if got.size else 0.0
