"""Debug the extreme-scales case: worst entries per fold vs the long-double truth."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle
from paper_2401_13185_b200 import cvgram as cv

rng = np.random.default_rng(11)
n, k, m, p = 6000, 70, 4, 7
x = rng.normal(0, 1, (n, k)) + rng.uniform(-5, 5, k)
x[:, 0] = 1e150 * (rng.normal(0, 1, n) + 3)
x[:, 1] = 1e-150 * (rng.normal(0, 1, n) - 2)
x[:, 2] = np.where(rng.random(n) < 0.5, -1.0, 1.0) * 63.0
x[:, 3] = 7.0
spike = rng.integers(n)
x[spike, 3] = 7.5
x[:, 4] = rng.standard_cauchy(n)
x[:, 5] = -2.5
x[:, 6] = np.where(rng.random(n) < 0.5, -1.0, 1.0) * (1 - 2.0 ** -40)
y = x[:, 7:11] @ rng.normal(0, 1, (4, m)) + rng.normal(0, 0.1, (n, m))
y[:, 0] = 1e120 * rng.normal(0, 1, n)
lab = (rng.permutation(n) % p + 1).astype(np.int32)
print("spike row", spike, "fold", lab[spike])
from test_gpu_parity import _transformed_norms
for cfg in (15,):
    got = cv.run_all_folds_configs(cv.DatasetPair(x, y), cv.Partitioning(lab, p), [cfg])[0]
    truth = oracle.truth_all_folds(x, y, lab, p, cfg, n_threads=8)
    for g, r in zip(got, truth):
        nx, nxc, ny = _transformed_norms(x, y, lab, r.fold_id, cfg, r)
        t = lab != r.fold_id
        rx = np.linalg.norm(x[t].astype(np.float64), axis=0)
        den = np.maximum(np.maximum(np.abs(r.xtx_t), np.outer(nx, nx)), 1e-8 * np.outer(rx, rx))
        e = np.abs(g.xtx_t - r.xtx_t) / np.where(den == 0, 1, den)
        i, j = np.unravel_index(np.argmax(e), e.shape)
        print(f"fold {r.fold_id}: worst {e[i, j]:.3e} at ({i},{j}) got {g.xtx_t[i, j]:.6e} truth {r.xtx_t[i, j]:.6e} "
              f"den {den[i, j]:.3e} nx {nx[i]:.3e} {nx[j]:.3e} rx {rx[i]:.3e} {rx[j]:.3e} sd_got {g.stats.std_x_t[i]:.6e} sd_ref {r.std_x_t[i]:.6e}")
