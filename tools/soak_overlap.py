"""Soak: the default schedule (cut beside the Gram, split last round) against the serial, unsplit schedule at the
full BASELINE sizes, many iterations, every output compared bit for bit (a cross-proxy or ordering race in the
per-segment publish / acquire protocol would show up as a rare mismatch).
usage: python tools/soak_overlap.py [--configs 1,2,4] [--iters 100]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import workloads
    from paper_2401_13185_b200 import plan as P

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4")
    ap.add_argument("--iters", type=int, default=100)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    for cid in [int(v) for v in a.configs.split(",")]:
        if cid in (3, 4):
            x, y, lab, p, cfgs = workloads.make_device(cid, dev)
        else:
            w = workloads.make(cid)
            x, y = torch.from_numpy(w.x).to(dev), torch.from_numpy(w.y).to(dev)
            lab, p, cfgs = torch.from_numpy(w.labels).to(dev), w.p, w.cfgs
        n, k = x.shape
        pl = P.DevicePlan(n, k, y.shape[1], p)
        os.environ["CVG_I8_OVERLAP"] = "0"
        os.environ["CVG_I8_SPLIT"] = "0"
        _, ref = P.run_all_folds_device(x, y, lab, p, list(cfgs), group=None, plan=pl)
        ref = {key: val.clone() for key, val in ref.items()}
        del os.environ["CVG_I8_OVERLAP"], os.environ["CVG_I8_SPLIT"]
        bad = 0
        for it in range(a.iters):
            _, out = P.run_all_folds_device(x, y, lab, p, list(cfgs), group=None, plan=pl)
            torch.cuda.synchronize()
            ok = all(torch.equal(out[key], ref[key]) for key in ref)
            bad += 0 if ok else 1
        print(json.dumps({"config": cid, "iters": a.iters, "mismatches": bad}), flush=True)
        del x, y, pl, ref, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
