"""numpy/OpenBLAS restatement of the reference's Algorithm 7 -- TEST / BASELINE INFRASTRUCTURE ONLY.

The second CPU point of BASELINE.md §2: the same computation as R64
(cvgram_oracle.c) with numpy's fp64 GEMM (OpenBLAS, all host threads) doing the
products.  Only bench.py's cpu_baseline leg times it; tests check it against R64.

Follows /root/reference/proj/include/cvgram/fast.hpp:
  precompute_global   fast.hpp:19-36  (XᵀX, XᵀY, sums, means, sums of squares)
  training_mean       fast.hpp:40-47  (from means, not from sums)
  training_std        fast.hpp:53-69  (reciprocal-scaled radicand, clamp, exact 0 -> 1)
  fold_products       fast.hpp:73-130 (gather, downdate, outer-then-times-n_t, divide by the product)
  run_all_folds       fast.hpp:133-152 (one configuration per call, folds in ascending order)
"""
from __future__ import annotations

import numpy as np


def _training_mean(g, v, n, nv):
    nt = float(n - nv)
    return (float(n) / nt) * g - (float(nv) / nt) * v


def _training_std(mean_t, sum_t, sum_sq_t, nt):
    scale = 1.0 / float(nt - 1)
    rad = scale * ((-2.0 * mean_t * sum_t + float(nt) * mean_t * mean_t) + sum_sq_t)
    sd = np.sqrt(np.maximum(rad, 0.0))
    return np.where(sd == 0.0, 1.0, sd)


def run_all_folds(x, y, labels, p, cfg):
    """All folds of one configuration; returns [(xtx_t, xty_t)] in fold order."""
    cx, cy, sx, sy = bool(cfg & 8), bool(cfg & 4), bool(cfg & 2), bool(cfg & 1)
    any_cfg, any_scale = cfg != 0, sx or sy
    n = x.shape[0]
    xtx, xty = x.T @ x, x.T @ y
    if any_cfg:
        sum_x, sum_y = x.sum(0), y.sum(0)
        mean_x, mean_y = sum_x / n, sum_y / n
    if any_scale:
        sq_x, sq_y = (x * x).sum(0), (y * y).sum(0)
    order = np.argsort(labels, kind="stable")  # build_validation_partitions: ascending rows per fold
    bounds = np.searchsorted(labels[order], np.arange(1, p + 2))
    out = []
    for f in range(p):
        v = order[bounds[f]:bounds[f + 1]]
        nv = v.size
        nt = n - nv
        xv, yv = x[v], y[v]
        gx, gy = xtx - xv.T @ xv, xty - xv.T @ yv
        if any_cfg:
            mx = _training_mean(mean_x, xv.sum(0) / nv, n, nv)
            my = _training_mean(mean_y, yv.sum(0) / nv, n, nv)
        if cx:
            gx = gx - float(nt) * np.outer(mx, mx)
        if cx or cy:
            gy = gy - float(nt) * np.outer(mx, my)
        if sx:
            sdx = _training_std(mx, sum_x - xv.sum(0), sq_x - (xv * xv).sum(0), nt)
            gx = gx / np.outer(sdx, sdx)
        if sy:
            sdy = _training_std(my, sum_y - yv.sum(0), sq_y - (yv * yv).sum(0), nt)
        if any_scale:
            gy = gy / np.outer(sdx if sx else np.ones(x.shape[1]), sdy if sy else np.ones(y.shape[1]))
        out.append((gx, gy))
    return out
