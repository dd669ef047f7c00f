"""Time one rank's step of a world-G run of BASELINE configs[1] on ONE GPU (no collective: the other ranks'
partials are stand-ins), to see how the per-rank work shrinks with G: which parts of the step do not scale.
usage: python tools/rank_emulation.py [--config 1] [--worlds 1,2,4,8]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import workloads
    from paper_2401_13185_b200 import _lib as L
    from paper_2401_13185_b200 import cvgram as cv
    from paper_2401_13185_b200 import plan as P

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = workloads.make(a.config)
    x, y = torch.from_numpy(w.x).to(dev), torch.from_numpy(w.y).to(dev)
    lab = torch.from_numpy(w.labels).to(dev)
    ctx = cv.get_context(0)
    stream = torch.cuda.current_stream(dev)
    ctx.use_torch_stream(stream)
    shift = torch.cat([x[0], y[0]]).double().cpu().numpy()
    names = ["bucket", "reorder", "gram", "tree_sum", "fold_stats", "products"]
    for world in [int(v) for v in a.worlds.split(",")]:
        for rank in sorted({0, world - 1}):
            pl = P.DevicePlan(w.n, w.k, w.m, w.p, ctx=ctx, rank=rank, world=world)
            gathered = torch.zeros(world * pl.partial_count, dtype=torch.float64, device=dev)
            mine = torch.empty(pl.partial_count, dtype=torch.float64, device=dev)
            out = None

            def step():
                nonlocal out
                pl.bind_labels(lab, True)
                pl.gram(x, y, shift)
                if world > 1:
                    pl.partial_into(mine)
                    gathered[rank * pl.partial_count:(rank + 1) * pl.partial_count].copy_(mine)
                    out = pl.finish(list(w.cfgs), gathered, world, out)
                else:
                    out = pl.finish(list(w.cfgs), None, 1, out)

            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            L.lib().cvg_context_enable_timing(ctx.handle, 1)
            for _ in range(a.steps):
                step()
            torch.cuda.synchronize()
            t, c = np.zeros(6), np.zeros(6, np.int64)
            L.lib().cvg_context_kernel_times(ctx.handle, t.ctypes.data, c.ctypes.data)
            L.lib().cvg_context_enable_timing(ctx.handle, 0)
            print(json.dumps({"config": a.config, "world": world, "rank": rank, "folds": pl.n_owned,
                              "ms_per_step": round(ms, 4),
                              "kernels_ms": {n: round(float(v) / a.steps, 4) for n, v in zip(names, t)}}), flush=True)


if __name__ == "__main__":
    main()
