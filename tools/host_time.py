"""Host-side time of the three plan calls of a device-resident pass (bind_labels, gram, finish): how much of
a small problem's step is host work (launches, tensor-map encodes, syncs) rather than kernels.
usage: python tools/host_time.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import workloads
    from paper_2401_13185_b200 import cvgram as cv
    from paper_2401_13185_b200 import plan as P

    dev = torch.device("cuda", 0)
    for cid in (0, 1):
        w = workloads.make(cid)
        x, y = torch.from_numpy(w.x).to(dev), torch.from_numpy(w.y).to(dev)
        lab = torch.from_numpy(w.labels).to(dev)
        pl = P.DevicePlan(w.n, w.k, w.m, w.p, ctx=cv.get_context(0))
        shift = torch.cat([x[0], y[0]]).double().cpu().numpy()
        masks = list(w.cfgs)
        out = None

        def phases():
            nonlocal out
            t0 = time.perf_counter()
            pl.bind_labels(lab, True)
            t1 = time.perf_counter()
            pl.gram(x, y, shift)
            t2 = time.perf_counter()
            out = pl.finish(masks, None, 1, out)
            t3 = time.perf_counter()
            return t1 - t0, t2 - t1, t3 - t2

        for _ in range(5):
            phases()
        acc = np.zeros(3)
        reps = 50
        for _ in range(reps):
            acc += np.array(phases())
        print(f"c{cid}: host ms per call (bind_labels, gram, finish) {np.round(acc / reps * 1e3, 4)}, "
              f"total {acc.sum() / reps * 1e3:.4f}", flush=True)


if __name__ == "__main__":
    main()
