"""The multi-GPU exchange protocol on CPU: world_size 2 and 4 over gloo.

Each rank owns its canonical fold range (cvg_fold_range), computes its
fold-tree node, all-gathers it (the run's one collective) and finishes its own
folds.  The per-rank compute is a numpy stand-in with the engine's structure
(shifted-basis fold Grams, midpoint-tree sums, the K5 formulas), injected via
``plan_factory``; what is under test is the product's driver
(plan.run_all_folds_device / exchange_partials / fold_range): that every fold
is produced exactly once, by the right rank, bit-identical to world_size 1 and
within 1e-10 of the long-double oracle.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _tree(vals, a, b):
    if b <= a:
        return np.zeros_like(vals[0]) if vals else 0.0
    if b - a == 1:
        return vals[a]
    mid = a + (b - a) // 2
    return _tree(vals, a, mid) + _tree(vals, mid, b)


class NumpyPlan:
    """CPU stand-in for DevicePlan with the engine's reduction structure."""

    def __init__(self, n, k, m, p, fb, fe):
        self.n, self.k, self.m, self.p, self.fold_begin, self.fold_end = n, k, m, p, fb, fe
        self.w = k + m
        self.partial_count = k * (self.w + 1)

    def bind_labels(self, labels, require_scalable):
        self.labels = labels.numpy()

    def gram(self, x, y, shift, row_map=None):
        z = np.concatenate([x.numpy(), y.numpy()], axis=1)
        if row_map is not None:  # compacted rows: rebuild the full row space (absent rows stay 0)
            rm = row_map.numpy()
            full = np.zeros((self.n, z.shape[1]))
            full[rm >= 0] = z[rm[rm >= 0]]
            assert np.all(rm[np.isin(self.labels, np.arange(self.fold_begin + 1, self.fold_end + 1))] >= 0)
            z = full
        self.shift = z[0].copy() if shift is None else np.asarray(shift)
        z = z - self.shift
        z1 = np.concatenate([z, np.ones((z.shape[0], 1))], axis=1)
        self.G = []
        for f in range(self.fold_begin, self.fold_end):
            zf = z1[self.labels == f + 1]
            self.G.append(zf.T @ zf)  # (w+1) x (w+1): sums in the ones column
        self.counts = np.bincount(self.labels, minlength=self.p + 1)[1:]
        w1 = self.w + 1
        self.local = _tree(self.G, 0, len(self.G)) if self.G else np.zeros((w1, w1))

    def partial_into(self, dst):
        dst.copy_(torch.from_numpy(np.ascontiguousarray(self.local[: self.k]).ravel()))

    def finish(self, masks, gathered=None, world=1, out=None):
        k, w = self.k, self.w
        if gathered is None:
            total_k = self.local[:k]
        else:
            g = gathered.numpy().reshape(world, k, w + 1)
            total_k = _tree([g[r] for r in range(world)], 0, world)
        full = self.local.copy()
        full[:k] = total_k
        res = {"xtx": [], "xty": []}
        for mask in masks:
            cx, cy, sx, sy = bool(mask & 8), bool(mask & 4), bool(mask & 2), bool(mask & 1)
            xx, xy = [], []
            for i, f in enumerate(range(self.fold_begin, self.fold_end)):
                G = self.G[i]
                nt = float(self.n - self.counts[f])
                T = total_k
                gt = T[:, :w] - G[:k, :w]
                sT = T[:, w] - G[:k, w]
                c = self.shift[:k]
                mz = sT / nt
                # Y-side sums / squares come from each rank's own data (same rows everywhere here)
                v = gt.copy()
                if cx:
                    v[:, :k] = gt[:, :k] - nt * np.outer(mz, mz)
                else:
                    v[:, :k] = gt[:, :k] + np.outer(c, sT) + np.outer(sT, c) + nt * np.outer(c, c)
                xx.append(v[:, :k])
                xy.append(v[:, k:])
            res["xtx"].append(np.stack(xx) if xx else np.zeros((0, k, k)))
            res["xty"].append(np.stack(xy) if xy else np.zeros((0, k, self.m)))
        return res


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir, data):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_13185_b200 import plan as P

    x, y, labels, p = data
    pl, out = P.run_all_folds_device(torch.from_numpy(x), torch.from_numpy(y), torch.from_numpy(labels), p, [8, 0],
                                     plan_factory=NumpyPlan)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), fb=pl.fold_begin, fe=pl.fold_end,
             xtx=np.stack(out["xtx"]), xty=np.stack(out["xty"]))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, data):
    with tempfile.TemporaryDirectory() as d:
        if world == 1:
            _worker_single(d, data)
        else:
            mp.spawn(_worker, args=(world, _free_port(), d, data), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        return [(int(q["fb"]), int(q["fe"]), q["xtx"], q["xty"]) for q in parts]


def _worker_single(d, data):
    from paper_2401_13185_b200 import plan as P

    x, y, labels, p = data
    pl, out = P.run_all_folds_device(torch.from_numpy(x), torch.from_numpy(y), torch.from_numpy(labels), p, [8, 0],
                                     plan_factory=NumpyPlan)
    np.savez(os.path.join(d, "rank0.npz"), fb=pl.fold_begin, fe=pl.fold_end, xtx=np.stack(out["xtx"]),
             xty=np.stack(out["xty"]))


@pytest.fixture(scope="module")
def data():
    rng = np.random.default_rng(11)
    n, k, m, p = 600, 9, 3, 7
    x = rng.normal(rng.uniform(-5, 5, k), rng.uniform(0.5, 2, k), (n, k))
    y = rng.normal(1, 1, (n, m))
    labels = rng.integers(1, p + 1, n).astype(np.int32)
    labels[:p] = np.arange(1, p + 1)
    return x, y, labels, p


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_cover_folds_and_match_world1_bitwise(world, data):
    single = _run(1, data)[0]
    parts = _run(world, data)
    covered = []
    for fb, fe, xtx, xty in parts:
        covered += list(range(fb, fe))
        assert np.array_equal(xtx, single[2][:, fb:fe]), f"world {world} folds {fb}:{fe}"
        assert np.array_equal(xty, single[3][:, fb:fe])
    assert covered == list(range(data[3]))


def test_world1_matches_long_double_oracle(data):
    import oracle

    x, y, labels, p = data
    fb, fe, xtx, xty = _run(1, data)[0]
    for ci, cfg in enumerate([8, 0]):
        truth = oracle.truth_all_folds(x, y, labels, p, cfg)
        for f in range(p):
            d = np.sqrt(np.abs(np.diag(truth[f].xtx_t)))
            err = np.abs(xtx[ci, f] - truth[f].xtx_t) / np.maximum(np.abs(truth[f].xtx_t), np.outer(d, d))
            assert err.max() <= 1e-10


def _worker_sharded(rank, world, port, outdir, data):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_13185_b200 import plan as P

    x, y, labels, p = data
    lo, hi = P.shard_rows(len(x), rank, world)
    pl, out = P.run_all_folds_sharded(torch.from_numpy(x[lo:hi]), torch.from_numpy(y[lo:hi]),
                                      torch.from_numpy(labels), p, [8, 0], n=len(x), plan_factory=NumpyPlan,
                                      device=torch.device("cpu"), exchange=os.environ.get("CVG_TEST_EXCHANGE", "auto"))
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), fb=pl.fold_begin, fe=pl.fold_end,
             xtx=np.stack(out["xtx"]), xty=np.stack(out["xty"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("exchange", ["alltoall", "allgather"])
def test_row_sharded_host_ingest_matches_world1_bitwise(world, exchange, data, monkeypatch):
    """run_all_folds_sharded: each rank holds only rows shard_rows(n, r, G) on
    the host.  alltoall: rows go only to their fold's owner and the plan reads
    them through a row map; allgather: every rank gets every row.  Either way:
    same folds, same bits as one rank (world 3 leaves a short last shard)."""
    monkeypatch.setenv("CVG_TEST_EXCHANGE", exchange)
    single = _run(1, data)[0]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_sharded, args=(world, _free_port(), d, data), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    covered = []
    for q in parts:
        fb, fe = int(q["fb"]), int(q["fe"])
        covered += list(range(fb, fe))
        assert np.array_equal(q["xtx"], single[2][:, fb:fe])
        assert np.array_equal(q["xty"], single[3][:, fb:fe])
    assert covered == list(range(data[3]))


def test_shard_rows_partition():
    from paper_2401_13185_b200 import plan as P

    for n in (1, 7, 600, 1001):
        for world in (1, 2, 3, 8):
            spans = [P.shard_rows(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


# ------------------------------------------------------------ the real CUDA rank plans, world 2 on one GPU
def _worker_cuda(rank, world, port, outdir, data):
    """A real DevicePlan per process (all on cuda:0); the partial Gram exchanged through host gloo -- no kernel
    waits on another process's kernel."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_13185_b200 import plan as P

    x, y, labels, p = data
    dev = torch.device("cuda", 0)
    pl = P.DevicePlan(x.shape[0], x.shape[1], y.shape[1], p, rank=rank, world=world)
    pl.bind_labels(torch.from_numpy(labels).to(dev), True)
    pl.gram(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
    mine = torch.empty(pl.partial_count, dtype=torch.float64, device=dev)
    pl.partial_into(mine)
    parts = [torch.empty(pl.partial_count, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, mine.cpu())
    out = pl.finish([15, 0], torch.cat(parts).to(dev), world)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), fb=pl.fold_begin, fe=pl.fold_end,
             xtx=out["xtx"].cpu().numpy(), xty=out["xty"].cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_cuda_rank_plans_over_gloo_match_single_gpu_bitwise(world):
    from paper_2401_13185_b200 import plan as P

    rng = np.random.default_rng(5)
    n, k, m, p = 30000, 70, 5, 6
    x = rng.normal(rng.uniform(-5, 5, k), rng.uniform(0.5, 2, k), (n, k))
    y = rng.normal(1, 1, (n, m))
    labels = (rng.permutation(n) % p + 1).astype(np.int32)
    dev = torch.device("cuda", 0)
    one = P.DevicePlan(n, k, m, p)
    one.bind_labels(torch.from_numpy(labels).to(dev), True)
    one.gram(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
    ref = one.finish([15, 0])
    rxx, rxy = ref["xtx"].cpu().numpy(), ref["xty"].cpu().numpy()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_cuda, args=(world, _free_port(), d, (x, y, labels, p)), nprocs=world, join=True)
        covered = []
        for r in range(world):
            q = np.load(os.path.join(d, f"rank{r}.npz"))
            fb, fe = int(q["fb"]), int(q["fe"])
            covered += list(range(fb, fe))
            assert np.array_equal(q["xtx"], rxx[:, fb:fe]) and np.array_equal(q["xty"], rxy[:, fb:fe])
        assert sorted(covered) == list(range(p))
