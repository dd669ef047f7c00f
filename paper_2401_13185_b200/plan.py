"""Device-resident staged engine (cvg_plan_*) and the multi-GPU driver.

A plan owns a contiguous fold range [fold_begin, fold_end) that is a node of
the canonical fold-sum tree (``fold_range``).  One process per GPU:

    bind_labels -> gram -> partial --all_gather (NCCL)--> finish

Only the partial (kp x kp doubles: the owned folds' shifted-basis Gram with
column sums and sums of squares riding in the ones column) crosses GPUs —
one collective per run, as the north star prescribes.  The all-gather + fixed
tree combine (instead of a rank-count-dependent all-reduce order) keeps
results bit-identical for 1, 2, 4 and 8 GPUs.

From host memory (``run_all_folds_sharded``) each rank copies only its row
shard over PCIe and the rows cross NVLink once: an all-to-all to their fold's
owner (the rank plan then reads compacted rows through a row map,
cvg_plan_gram_mapped), or an all-gather when folds are shared (P < G).
``DevicePlan.iter_folds`` streams the emitted folds in batches
(cvg_plan_finish_range) for leave-one-out-scale P.

PyTorch is plumbing here: device buffers, the current stream, and
torch.distributed for the collectives.  No torch types cross the C ABI.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from .cvgram import Context, PreprocessConfig, _cfg, _check, get_context


def fold_range(p: int, rank: int, world: int):
    """Canonical folds [begin, end) of `rank` among `world` (cvg_fold_range)."""
    b, e = ctypes.c_int32(), ctypes.c_int32()
    rc = L.lib().cvg_fold_range(p, rank, world, ctypes.addressof(b), ctypes.addressof(e))
    if rc != L.OK:
        raise ValueError(f"invalid fold_range({p}, {rank}, {world})")
    return b.value, e.value


def _dptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


class DevicePlan:
    """Thin owner of a cvg_plan; arguments are torch CUDA tensors.

    Either an explicit fold range, or ``rank``/``world``: the canonical fold-
    tree node is then chosen at bind time (shared folds when world > p) and
    ``fold_begin``/``fold_end`` give the folds this plan emits.
    """

    def __init__(self, n: int, k: int, m: int, p: int, fold_begin: int = 0, fold_end: Optional[int] = None,
                 dtype: str = "f64", ctx: Optional[Context] = None, rank: Optional[int] = None,
                 world: Optional[int] = None):
        import torch

        self.ctx = ctx or get_context()
        self.n, self.k, self.m, self.p = n, k, m, p
        self.fold_begin = fold_begin
        self.fold_end = p if fold_end is None else fold_end
        self.dtype_code = L.DTYPE_F32 if dtype in ("f32", "float32", torch.float32) else L.DTYPE_F64
        self.ctx.use_torch_stream(torch.cuda.current_stream(self.ctx.device))
        h = ctypes.c_void_p()
        buf = L.err_buf()
        if rank is not None:
            _check(L.lib().cvg_plan_create_rank(self.ctx.handle, self.dtype_code, n, k, m, p, rank, world,
                                                ctypes.byref(h), buf, len(buf)), buf)
        else:
            _check(L.lib().cvg_plan_create(self.ctx.handle, self.dtype_code, n, k, m, p, self.fold_begin,
                                           self.fold_end, ctypes.byref(h), buf, len(buf)), buf)
        self._h = h
        import weakref

        self._fin = weakref.finalize(self, L.lib().cvg_plan_destroy, h)
        cnt = ctypes.c_int64()
        L.lib().cvg_plan_partial(self._h, None, ctypes.byref(cnt))
        self.partial_count = int(cnt.value)

    @property
    def n_owned(self) -> int:
        return self.fold_end - self.fold_begin

    def bind_labels(self, labels, require_scalable: bool) -> None:
        buf = L.err_buf()
        _check(L.lib().cvg_plan_bind_labels(self._h, _dptr(labels), int(require_scalable), buf, len(buf)), buf)
        b, e = ctypes.c_int32(), ctypes.c_int32()
        L.lib().cvg_plan_assignment(self._h, ctypes.addressof(b), ctypes.addressof(e))
        self.fold_begin, self.fold_end = b.value, e.value

    def gram(self, x, y, shift: Optional[np.ndarray] = None, row_map=None) -> None:
        """row_map (int64 CUDA tensor, n entries): x / y are compacted, original
        row i at row_map[i] (-1 = absent); shift is then required."""
        buf = L.err_buf()
        sh = None if shift is None else np.ascontiguousarray(shift, np.float64)
        if row_map is not None:
            if sh is None:
                raise ValueError("a row-mapped gram needs an explicit shift")
            _check(L.lib().cvg_plan_gram_mapped(self._h, _dptr(x), x.stride(0), _dptr(y), y.stride(0),
                                                _dptr(row_map), x.shape[0], sh.ctypes.data, buf, len(buf)), buf)
            return
        _check(L.lib().cvg_plan_gram(self._h, _dptr(x), x.stride(0), _dptr(y), y.stride(0),
                                     None if sh is None else sh.ctypes.data, buf, len(buf)), buf)

    def partial_into(self, dst) -> None:
        cnt = ctypes.c_int64()
        rc = L.lib().cvg_plan_partial(self._h, _dptr(dst), ctypes.byref(cnt))
        if rc != L.OK:
            raise RuntimeError("cvg_plan_partial failed")

    def finish(self, cfg_masks: Sequence[int], rank_partials=None, n_ranks: int = 1, out=None):
        import torch

        dev = torch.device("cuda", self.ctx.device)
        masks = np.ascontiguousarray(cfg_masks, np.uint32)
        nc, no, k, m = masks.size, self.n_owned, self.k, self.m
        if out is None:
            f64 = torch.float64
            out = {"xtx": torch.empty((nc, no, k, k), dtype=f64, device=dev),
                   "xty": torch.empty((nc, no, k, m), dtype=f64, device=dev),
                   "mean_x": torch.empty((no, k), dtype=f64, device=dev),
                   "mean_y": torch.empty((no, m), dtype=f64, device=dev),
                   "std_x": torch.empty((no, k), dtype=f64, device=dev),
                   "std_y": torch.empty((no, m), dtype=f64, device=dev)}
        buf = L.err_buf()
        _check(L.lib().cvg_plan_finish(self._h, _dptr(rank_partials), n_ranks, masks.ctypes.data, nc,
                                       _dptr(out["xtx"]), _dptr(out["xty"]), _dptr(out.get("mean_x")),
                                       _dptr(out.get("mean_y")), _dptr(out.get("std_x")), _dptr(out.get("std_y")),
                                       buf, len(buf)), buf)
        return out

    def finish_range(self, cfg_masks: Sequence[int], fold_lo: int, fold_hi: int, rank_partials=None,
                     n_ranks: int = 1, out=None):
        """finish() for emitted folds [fold_lo, fold_hi) only; outputs packed for the range."""
        import torch

        dev = torch.device("cuda", self.ctx.device)
        masks = np.ascontiguousarray(cfg_masks, np.uint32)
        nc, nf, k, m = masks.size, fold_hi - fold_lo, self.k, self.m
        if out is None or out["xtx"].shape[1] != nf or out["xtx"].shape[0] != nc:
            f64 = torch.float64
            out = {"xtx": torch.empty((nc, nf, k, k), dtype=f64, device=dev),
                   "xty": torch.empty((nc, nf, k, m), dtype=f64, device=dev),
                   "mean_x": torch.empty((nf, k), dtype=f64, device=dev),
                   "mean_y": torch.empty((nf, m), dtype=f64, device=dev),
                   "std_x": torch.empty((nf, k), dtype=f64, device=dev),
                   "std_y": torch.empty((nf, m), dtype=f64, device=dev)}
        view = out
        buf = L.err_buf()
        _check(L.lib().cvg_plan_finish_range(self._h, _dptr(rank_partials), n_ranks, masks.ctypes.data, nc, fold_lo,
                                             fold_hi, _dptr(view["xtx"]), _dptr(view["xty"]),
                                             _dptr(view["mean_x"]), _dptr(view["mean_y"]), _dptr(view["std_x"]),
                                             _dptr(view["std_y"]), buf, len(buf)), buf)
        return view

    def iter_folds(self, cfg_masks: Sequence[int], batch: int, rank_partials=None, n_ranks: int = 1):
        """Stream the emitted folds in batches of `batch` (lazy per-fold generation:
        leave-one-out-scale P without P x K x K of outputs in memory).  Yields
        (fold_lo, fold_hi, outputs) with device tensors reused between batches."""
        out = None
        for lo in range(self.fold_begin, self.fold_end, batch):
            hi = min(lo + batch, self.fold_end)
            out = self.finish_range(cfg_masks, lo, hi, rank_partials, n_ranks, out)  # reallocated only if shorter
            yield lo, hi, out

    def fold_counts(self) -> np.ndarray:
        c = np.empty(self.p, np.int64)
        L.lib().cvg_plan_fold_counts(self._h, c.ctypes.data)
        return c


def run_all_folds_device(x, y, labels, p: int, cfgs, group=None, plan=None, shift: Optional[np.ndarray] = None,
                         plan_factory=None):
    """All folds of `labels` on device-resident x/y/labels (torch CUDA tensors).

    With a torch.distributed process group of size G > 1, this rank computes
    only its canonical fold range and the ranks exchange one partial Gram by
    all-gather.  Returns (plan, outputs) where outputs hold the owned folds.
    Every rank must pass the same `shift` (default: row 0 of the full x | y).
    `plan_factory(n, k, m, p, fold_begin, fold_end)` substitutes the plan
    object (tests drive this exchange logic on CPU with gloo).
    """
    import torch
    import torch.distributed as dist

    cfgs = [_cfg(c) for c in cfgs]
    masks = [c.mask for c in cfgs]
    distributed = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if distributed else 1
    rank = dist.get_rank(group) if distributed else 0
    n, k = x.shape
    m = y.shape[1]
    if plan is None:
        if plan_factory is not None:
            fb, fe = fold_range(p, rank, world)
            plan = plan_factory(n, k, m, p, fb, fe)
        else:
            plan = DevicePlan(n, k, m, p, dtype="f32" if x.dtype == torch.float32 else "f64", rank=rank, world=world)
    plan.bind_labels(labels, require_scalable=any(c.any_scale() for c in cfgs))
    plan.gram(x, y, shift)
    if world > 1:
        mine = torch.empty(plan.partial_count, dtype=torch.float64, device=x.device)
        plan.partial_into(mine)
        gathered = exchange_partials(mine, world, group)
        out = plan.finish(masks, gathered, world)
    else:
        out = plan.finish(masks)
    return plan, out


def shard_rows(n: int, rank: int, world: int):
    """Rows [lo, hi) of the row-sharded host ingest: blocks of ceil(n / world)
    rows in rank order (only the last shard is short)."""
    s = -(-n // world)
    return min(n, rank * s), min(n, (rank + 1) * s)


def fold_owners(p: int, world: int):
    """Rank owning each fold (0-based) when every rank owns whole folds (p >= world), else None."""
    if p < world:
        return None
    own = np.empty(p, np.int64)
    for r in range(world):
        b, e = fold_range(p, r, world)
        own[b:e] = r
    return own


def run_all_folds_sharded(x_shard, y_shard, labels, p: int, cfgs, n: int, group=None, plan=None,
                          plan_factory=None, device=None, out_host=None, gather: Optional[bool] = None,
                          exchange: str = "auto"):
    """Multi-GPU entry point from HOST memory (the e2e path at N GPUs).

    This rank holds rows ``shard_rows(n, rank, world)`` of x | y in host memory
    (pinned for full PCIe speed) and all n labels.  Each rank copies only its
    shard over its own PCIe link; the rows then move over NVLink:

    * ``alltoall`` (default when every rank owns whole folds, p >= world): each
      row goes only to the rank that owns its fold (one all_to_all per matrix,
      rows stably bucketed by owner, so each owner receives its folds' rows in
      original order); the plan reads the compacted rows through a row map
      (cvg_plan_gram_mapped).  Row 0 (the shift) is broadcast from rank 0.
    * ``allgather`` (p < world, shared folds): every rank receives every row.

    Either way the canonical fold-range run follows (one partial all-gather,
    the owned folds' epilogue), bit-identical to one GPU.  Returns (plan,
    outputs) with the owned folds' outputs copied to host tensors (``out_host``
    reused when given).  ``gather`` forces (or skips) the row exchange;
    default: only when world > 1.
    """
    import torch
    import torch.distributed as dist

    cfgs = [_cfg(c) for c in cfgs]
    masks = [c.mask for c in cfgs]
    distributed = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if distributed else 1
    rank = dist.get_rank(group) if distributed else 0
    lo, hi = shard_rows(n, rank, world)
    if x_shard.shape[0] != hi - lo or y_shard.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} must hold rows [{lo}, {hi}) of x and y")
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if torch.cuda.is_available() else torch.device("cpu"))
    k, m = x_shard.shape[1], y_shard.shape[1]
    s = -(-n // world)
    d_labels = labels.to(dev, non_blocking=True)
    do_exchange = (world > 1) if gather is None else (gather and distributed)
    owners = fold_owners(p, world) if do_exchange else None
    if exchange == "auto":
        exchange = "alltoall" if owners is not None else "allgather"
    if do_exchange and exchange == "alltoall" and owners is not None:
        mine_x = x_shard.to(dev, non_blocking=True)
        mine_y = y_shard.to(dev, non_blocking=True)
        lut = torch.from_numpy(owners).to(dev)
        lab0 = (d_labels.long() - 1).clamp(0, p - 1)  # out-of-range labels: the plan's bind reports them
        dest = lut[lab0[lo:hi]]
        dest_sorted, perm = torch.sort(dest, stable=True)
        send_counts = torch.bincount(dest_sorted, minlength=world)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=group)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        x = torch.empty((sum(rc), k), dtype=x_shard.dtype, device=dev)
        y = torch.empty((sum(rc), m), dtype=y_shard.dtype, device=dev)
        dist.all_to_all_single(x, mine_x.index_select(0, perm), output_split_sizes=rc, input_split_sizes=sc,
                               group=group)
        dist.all_to_all_single(y, mine_y.index_select(0, perm), output_split_sizes=rc, input_split_sizes=sc,
                               group=group)
        owned = lut[lab0] == rank
        row_map = torch.where(owned, torch.cumsum(owned.long(), 0) - 1, torch.full_like(lab0, -1))
        sh = torch.empty(k + m, dtype=torch.float64, device=dev)
        if rank == 0:
            sh.copy_(torch.cat([mine_x[0].double(), mine_y[0].double()]))
        dist.broadcast(sh, src=0, group=group)
        shift = sh.cpu().numpy()
        if plan is None:
            if plan_factory is not None:
                fb, fe = fold_range(p, rank, world)
                plan = plan_factory(n, k, m, p, fb, fe)
            else:
                plan = DevicePlan(n, k, m, p, dtype="f32" if x.dtype == torch.float32 else "f64", rank=rank,
                                  world=world)
        plan.bind_labels(d_labels, require_scalable=any(c.any_scale() for c in cfgs))
        if (plan.fold_begin, plan.fold_end) != fold_range(p, rank, world):
            raise RuntimeError("rank plan does not own its canonical fold range")
        plan.gram(x, y, shift, row_map=row_map)
        mine = torch.empty(plan.partial_count, dtype=torch.float64, device=dev)
        plan.partial_into(mine)
        out = plan.finish(masks, exchange_partials(mine, world, group), world)
    else:
        mine_x = torch.zeros((s, k), dtype=x_shard.dtype, device=dev)
        mine_y = torch.zeros((s, m), dtype=y_shard.dtype, device=dev)
        mine_x[: hi - lo].copy_(x_shard, non_blocking=True)
        mine_y[: hi - lo].copy_(y_shard, non_blocking=True)
        if do_exchange:
            if dist.get_backend(group) == "nccl":
                full_x = torch.empty((world * s, k), dtype=x_shard.dtype, device=dev)
                full_y = torch.empty((world * s, m), dtype=y_shard.dtype, device=dev)
                dist.all_gather_into_tensor(full_x, mine_x, group=group)
                dist.all_gather_into_tensor(full_y, mine_y, group=group)
            else:
                px = [torch.empty_like(mine_x) for _ in range(world)]
                py = [torch.empty_like(mine_y) for _ in range(world)]
                dist.all_gather(px, mine_x, group=group)
                dist.all_gather(py, mine_y, group=group)
                full_x, full_y = torch.cat(px), torch.cat(py)
            x, y = full_x[:n], full_y[:n]
        else:
            x, y = mine_x[:n], mine_y[:n]
        plan, out = run_all_folds_device(x, y, d_labels, p, cfgs, group=group, plan=plan, plan_factory=plan_factory)
    if not isinstance(out, dict) or not all(hasattr(v, "to") for v in out.values()):
        return plan, out  # stand-in plans (CPU tests) return host arrays already
    if out_host is None:
        out_host = {kk: torch.empty(v.shape, dtype=v.dtype, pin_memory=torch.cuda.is_available())
                    for kk, v in out.items()}
    for kk, v in out.items():
        out_host[kk].copy_(v, non_blocking=True)
    if dev.type == "cuda":
        torch.cuda.current_stream(dev).synchronize()
    return plan, out_host


def exchange_partials(mine, world: int, group=None):
    """The run's single collective: all-gather every rank's fold-tree node, in
    rank order (NCCL all_gather_into_tensor over NVLink; list form on gloo)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        gathered = torch.empty(world * mine.numel(), dtype=mine.dtype, device=mine.device)
        dist.all_gather_into_tensor(gathered, mine, group=group)
        return gathered
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return torch.cat(parts)

def gram_tiles(k: int, m: int, edge: int = 64):
    """Upper tiles the fold Gram computes (mirror of engine.cu gram_tiles)."""
    kp = -(-(k + m + 1) // edge) * edge
    nt, tx, to = kp // edge, (k - 1) // edge, (k + m) // edge
    return [(i, j) for i in range(nt) for j in range(i, nt) if i <= tx or j == i or j == to]


def fp64_kind() -> str:
    """The fp64 Gram kind plans are created with: "i8" (exact int8 digit slices on tcgen05 kind::i8,
    the default) or "dmma" (CVG_FP64_KIND=dmma: fp64 DMMA tiles)."""
    return "dmma" if os.environ.get("CVG_FP64_KIND") == "dmma" else "i8"


def i8_slices() -> int:
    return 5 if os.environ.get("CVG_I8_SLICES") == "5" else 6


def i8_pairs(s: int) -> int:
    """Slice pairs the int8 Gram multiplies: t + u <= s-1, plus the square (s/2, s/2) for even s."""
    return s * (s + 1) // 2 + (1 if s % 2 == 0 else 0)


def fp32_kind() -> str:
    """The fp32 Gram kind: "f16" (scaled fp16 hi/lo on kind::f16, default) or "tf32" (CVG_FP32_KIND=tf32)."""
    return "tf32" if os.environ.get("CVG_FP32_KIND") == "tf32" else "f16"


def executed_gram_flops(n: int, k: int, m: int, p: int, f32: bool = False) -> float:
    """Tensor-core flops the Gram kernel issues for n rows (fold padding ignored):
    fp64: 64x64 DMMA tiles, diagonal tiles only their 36 upper 8x8 blocks;
    fp32: 128x128 tcgen05 tiles x 3 products (fp16 hi/lo split by default, TF32 with CVG_FP32_KIND=tf32)."""
    if f32:
        return 3 * 2.0 * len(gram_tiles(k, m, 128)) * 128 * 128 * n
    tiles = gram_tiles(k, m)
    if fp64_kind() == "i8":  # int8 ops: 128x64 tiles x slice pairs
        tq = {(i // 2, j) for i, j in tiles}
        return 2.0 * len(tq) * 128 * 64 * n * i8_pairs(i8_slices())
    n_diag = sum(1 for i, j in tiles if i == j)
    return 2.0 * ((len(tiles) - n_diag) * 64 * 64 + n_diag * 36 * 64) * n
