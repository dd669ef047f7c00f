"""The paper's Fig. 1 sweep on one B200: time for all folds vs P (N=100,000, K=500, M=10, fp64,
balanced folds, P in {3, 5, 10, 100, 1000, 10000, 100000}), center+scale X and Y.

Device-resident inputs; per P: bind (device bucketing) + Gram + every fold's statistics and XtX / XtY, emitted in
batches of at most `--batch-gb` of output into reused device buffers (the reference API would hold all P folds
at once: 204 GB at P = N).  Times are CUDA events, min of --reps.

    python tools/p_sweep.py [--out profiles/r01_p_sweep.jsonl]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_13185_b200 import cvgram as cv  # noqa: E402
from paper_2401_13185_b200 import plan as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--k", type=int, default=500)
    ap.add_argument("--m", type=int, default=10)
    ap.add_argument("--p-list", default="3,5,10,100,1000,10000,100000")
    ap.add_argument("--batch-gb", type=float, default=8.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    n, k, m = args.n, args.k, args.m
    rng = cv.MT19937_64(42)
    data = cv.random_dataset(n, k, m, rng)  # random.hpp:19-33 (the reference's own generator)
    dev = torch.device("cuda", 0)
    xd, yd = torch.from_numpy(data.x()).to(dev), torch.from_numpy(data.y()).to(dev)
    lines = []
    for p in [int(t) for t in args.p_list.split(",")]:
        part = cv.random_partitioning(n, p, rng)  # random.hpp:38-50: balanced folds
        ld = torch.from_numpy(part.labels).to(dev)
        pl = P.DevicePlan(n, k, m, p)
        per_fold = (k * k + k * m) * 8
        batch = max(1, min(p, int(args.batch_gb * 1e9 // per_fold)))

        def run():
            pl.bind_labels(ld, True)
            pl.gram(xd, yd)
            for _lo, _hi, _out in pl.iter_folds([15], batch):
                pass

        run()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        line = {"n": n, "k": k, "m": m, "p": p, "cfg": "1111", "ms": round(best, 3),
                "folds_per_batch": batch, "output_gb": round(p * per_fold / 1e9, 2),
                "gflops_algorithmic": round(2.0 * n * k * (k + m) / (best * 1e-3) / 1e9, 1)}
        lines.append(line)
        print(json.dumps(line), flush=True)
        del pl
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            f.write("\n".join(json.dumps(x) for x in lines) + "\n")


if __name__ == "__main__":
    main()
