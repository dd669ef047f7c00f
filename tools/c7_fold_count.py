"""Acceptance criterion C7 on the B200 engine (acceptance.cpp:199-225): fold-count independence at desk scale.

N = 20,000, K = 100, M = 5, center + scale X and Y, data and labels from the reference's seeded generators
(random_dataset / random_partitioning, std::mt19937_64 seed 107).  Times the reference API call
run_all_folds (C ABI host entry: H2D of X | Y, every fold's outputs back in host memory) at P = 10 and
P = 1000 (min of 3, as min_wall_time), and the baseline engine (direct definition, baseline.hpp; on the
device) at the same P after a warm-up call (min of 3 at P = 10, 1 at P = 1000).  The reference's bars: fast(1000) <= 3 fast(10), base(1000) >= 20 base(10),
base(1000) >= 50 fast(1000).

    python tools/c7_fold_count.py [--out profiles/r02_c7.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_13185_b200 import cvgram as cv  # noqa: E402


def min_wall_time(reps, fn):
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    return best


def measure():
    rng = cv.MT19937_64(107)
    n, k, m = 20000, 100, 5
    data = cv.random_dataset(n, k, m, rng)
    cfg = cv.PreprocessConfig(True, True, True, True)
    part10 = cv.random_partitioning(n, 10, rng)
    part1000 = cv.random_partitioning(n, 1000, rng)
    cv.run_all_folds(data, part10, cfg)  # warm-up: context, kernels, pinned staging
    fast10 = min_wall_time(3, lambda: cv.run_all_folds(data, part10, cfg))
    fast1000 = min_wall_time(3, lambda: cv.run_all_folds(data, part1000, cfg))
    cv.baseline_fold_products(data, part10, cfg)  # warm-up: the baseline engine's first call loads its kernels
    base10 = min_wall_time(3, lambda: cv.baseline_fold_products(data, part10, cfg))
    base1000 = min_wall_time(1, lambda: cv.baseline_fold_products(data, part1000, cfg))
    return {"criterion": "C7 fold-count independence (acceptance.cpp:199-225)", "n": n, "k": k, "m": m,
            "fast10_s": fast10, "fast1000_s": fast1000, "base10_s": base10, "base1000_s": base1000,
            "fast_ratio": fast1000 / fast10, "base_ratio": base1000 / base10, "base_over_fast": base1000 / fast1000,
            "pass": fast1000 <= 3.0 * fast10 and base1000 >= 20.0 * base10 and base1000 >= 50.0 * fast1000}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    r = measure()
    line = json.dumps(r)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
