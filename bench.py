"""Benchmark of the all-fold CV XᵀX/XᵀY hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1]

Workload: BASELINE.json configs[1] (fp64, N=1e6, K=500, M=10, P=100 near-equal
folds, center+scale X and Y) -- the largest config quoted for one B200.  Both
arms generate the SAME host data (workloads.make: numpy generator + a numpy
std::mt19937_64 for the labels, no .so involved) and print the same `config`.

A step (ours) is one complete all-fold pass on the device: fold bucketing,
sampled segment maxima, K1Q (gather + shift + cut into 6 int8 digits), the
tcgen05 kind::i8 segmented fold Gram (exact integer slice products, fp64
drain), fixed-order fold sums, [all-gather of the partial Gram across ranks],
fold statistics + products for every configuration mask.

  value     algorithmic GFLOP/s (2·N·K(K+M) per step) with inputs resident in
            HBM, CUDA events on the engine stream, max over ranks.  Inputs are
            4.1 GB > 126 MB L2, so no L2 flush is needed between steps.
  e2e       the same metric through the reference-facing C ABI call
            cvg_run_all_folds with pinned HOST buffers: H2D of X, Y, labels and
            D2H of every fold's XᵀX/XᵀY and statistics inside the timed region.
  roofline  the Gram (dominant kernel): int8 tensor ops it issues per second
            against the measured tcgen05 kind::i8 issue-loop peak; the line also
            carries its fp64-equivalent rate against the measured FP64 (DMMA) peak.
  cpu_baseline  R64 (oracle/, fast.hpp Algorithm 7 in C, all host threads), min
            of 3 runs, plus the numpy/OpenBLAS Algorithm 7 point.

--impl reference times the reference algorithm's CPU restatement (R64; the C++
reference itself cannot be built here: Eigen3/Catch2/CLI11 are absent) on this
box's host cores over exactly --warmup + --steps steps of the same workload.
It never loads the engine library.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Measured on this pool's B200s (profiles/): the denominators of the roofline fractions.
FP64_DMMA_PEAK_TFLOPS = 37.1  # profiles/r01_fp64_peaks.txt: DMMA.8x8x4 issue loop (cuBLAS DGEMM 35.4)
TF32_PEAK_TFLOPS = 623.3      # profiles/r01_fp64_peaks.txt: cuBLAS TF32 8192^3 sustained
# tcgen05.mma kind::i8 issue loop (tools/i8_peak.cu, M=128 N=256 K=32, one CTA per SM, resident operands):
# profiles/r02_i8_peak.txt.  NVIDIA's nominal dense int8 figure is 4500 TOPS.
INT8_PEAK_TOPS = float(os.environ.get("CVG_INT8_PEAK_TOPS", "4500.0"))
INT8_PEAK_SOURCE = "NVIDIA nominal dense int8 (4.5 POPS)"
_PEAKS_R02 = os.path.join(ROOT, "profiles", "r02_i8_peak.json")
if os.path.exists(_PEAKS_R02) and "CVG_INT8_PEAK_TOPS" not in os.environ:
    try:
        _pk = json.load(open(_PEAKS_R02))
        INT8_PEAK_TOPS = float(_pk["tops"])
        INT8_PEAK_SOURCE = _pk["source"]
    except Exception:
        pass
CPU_SAMPLE_ROWS = 1_000_000
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--data", choices=["auto", "host", "device"], default="auto",
                    help="host: workloads.make (both arms' data); device: torch generator on the GPU "
                         "(auto: host for configs 0-2, device for the 16-23 GB configs 3-4)")
    ap.add_argument("--e2e-path", choices=["auto", "capi", "sharded"], default="auto",
                    help="auto: the C ABI call at N=1, the row-sharded host entry at N>1")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def host_cpu():
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count() or 1}


def use_host_data(cid, args):
    return args.data == "host" or (args.data == "auto" and cid in (0, 1, 2))


def bench_config(cid):
    """The `config` object both arms print (identical by construction)."""
    import workloads

    n, k, m, p = workloads.SHAPES[cid]
    return {"workload": f"configs[{cid}] N={n} K={k} M={m} P={p} cfg masks {workloads.CONFIGS[cid]} "
                        f"({workloads.DESCRIPTIONS[cid]})",
            "global_batch": n, "seed": workloads.SEEDS[cid],
            "input_dtype": "f64" if workloads.DTYPES[cid] == np.float64 else "f32",
            "parallelism": "folds across workers (GPU ranks | host threads)"}


# ------------------------------------------------------------- clock sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self.after = False
        if not self.lines:  # run shorter than nvidia-smi's start-up: one sample right after it
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=30)
                self.lines = [ln.strip() for ln in out.stdout.splitlines() if ln.strip()]
                self.after = bool(self.lines)
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
               "reasons": sorted(reasons), "samples": len(sm)}
        if getattr(self, "after", False):
            out["note"] = "timed region shorter than the sampler's start-up: sampled right after it"
        return out


# ------------------------------------------------------------- CPU arms
def cpu_sample(cid: int, sample_rows: int):
    import workloads

    n0 = workloads.SHAPES[cid][0]
    return workloads.make(cid, scale=min(1.0, sample_rows / n0))  # bounded sample, never larger than the config


def time_r64(w, warmup: int, steps: int):
    """R64 (oracle port of fast.hpp Algorithm 7) on all host threads; one run_all_folds call
    per configuration mask (the reference API serves one configuration per call)."""
    import oracle

    cores = os.cpu_count() or 1
    xd, yd = w.x.astype(np.float64), w.y.astype(np.float64)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        for cfg in w.cfgs:
            oracle.fast_all_folds(xd, yd, w.labels, w.p, cfg, n_threads=cores)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return times, cores


def time_numpy(w, reps: int):
    """numpy/OpenBLAS Algorithm 7 (oracle/numpy_alg7.py) on all host threads, min of `reps`."""
    from oracle import numpy_alg7

    xd, yd = w.x.astype(np.float64), w.y.astype(np.float64)
    best = float("inf")
    for _ in range(reps + 1):  # one warm-up
        t0 = time.perf_counter()
        for cfg in w.cfgs:
            numpy_alg7.run_all_folds(xd, yd, w.labels, w.p, cfg)
        best = min(best, time.perf_counter() - t0)
    return best


def r64_desc(w, cores, runs, how):
    return (f"configs[{w.cid}] workload with N={w.n} rows (seed {w.seed}), K={w.k}, M={w.m}, P={w.p}, cfg masks "
            f"{w.cfgs} (one run_all_folds call each); R64 = oracle/cvgram_oracle.c restating fast.hpp:19-152 "
            f"(blocked AVX fp64 GEMM; the global product and {cores} fold threads -- the reference runs its global "
            f"Eigen product on one thread, fast.hpp:23-24); {how} of {runs} runs")


def run_reference(args):
    """The reference arm: R64 on this box's host cores, exactly W warm-up + K timed steps."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cid = args.config
    w = cpu_sample(cid, CPU_SAMPLE_ROWS)
    flops = w.flops
    t0 = time.perf_counter()
    times, cores = time_r64(w, args.warmup, args.steps)
    total = time.perf_counter() - t0
    ms = 1e3 * sum(times) / len(times)
    value = flops / (ms * 1e-3) / 1e9
    cpu = host_cpu()
    line = {"impl": "reference", "metric": "all_fold_cv_gram_gflops", "value": round(value, 3),
            "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (workloads.make, host numpy; same as --impl ours)",
            "config": bench_config(cid),
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores, "kind": "port",
                             "sample": r64_desc(w, cores, len(times), "mean") + (
                                 "" if w.n == workloads_n(cid) else f" (bounded sample of {w.n} rows, "
                                 "GFLOP/s scaled by its own 2NK(K+M))"),
                             "min_ms": round(1e3 * min(times), 3), "host": cpu},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "timed_region_s": round(sum(times), 3), "run_s": round(total, 3),
            "note": "reference C++ (Eigen3/Catch2/CLI11) cannot be built in this image; the oracle restatement of "
                    "its algorithm (R64) is timed instead, W warm-up + K timed steps exactly as declared"}
    print(json.dumps(line), flush=True)


def workloads_n(cid):
    import workloads

    return workloads.SHAPES[cid][0]


# ---------------------------------------------------------------- our arm
def relaunch_distributed(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: launch N ranks ourselves (one process per GPU)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def run_ours(args):
    import torch
    import torch.distributed as dist

    import workloads
    from paper_2401_13185_b200 import _lib as L
    from paper_2401_13185_b200 import cvgram as cv
    from paper_2401_13185_b200 import plan as P

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = cv.get_context(local)
    cid = args.config
    n, k, m, p = workloads.SHAPES[cid]
    host = None
    if use_host_data(cid, args):
        host = workloads.make(cid)
        x = torch.from_numpy(host.x).to(dev)
        y = torch.from_numpy(host.y).to(dev)
        labels = torch.from_numpy(host.labels).to(dev)
        cfgs = host.cfgs
        data_note = "synthetic (workloads.make, host numpy; same as --impl reference)"
    else:
        x, y, labels, p, cfgs = workloads.make_device(cid, dev)
        data_note = "synthetic (workloads.make_device: the config's distributions drawn on the GPU with torch)"
    masks = list(cfgs)  # every configuration the BASELINE config names, from one Gram pass
    flops = 2.0 * n * k * (k + m)
    plan = P.DevicePlan(n, k, m, p, dtype="f32" if x.dtype == torch.float32 else "f64", ctx=ctx, rank=rank,
                        world=world)
    stream = torch.cuda.current_stream(dev)
    ctx.use_torch_stream(stream)

    # row 0 of the full data is every rank's shift
    shift = torch.cat([x[0], y[0]]).double().cpu().numpy()
    out = None
    mine = gathered = None
    if world > 1:
        mine = torch.empty(plan.partial_count, dtype=torch.float64, device=dev)
        gathered = torch.empty(world * plan.partial_count, dtype=torch.float64, device=dev)

    def step():
        nonlocal out
        plan.bind_labels(labels, True)
        plan.gram(x, y, shift)
        if world > 1:
            plan.partial_into(mine)
            dist.all_gather_into_tensor(gathered, mine)  # the run's single collective (NVLink)
            out = plan.finish(masks, gathered, world, out)
        else:
            out = plan.finish(masks, None, 1, out)

    clocks = ClockSampler(local).__enter__()  # sampled over warm-up + timed steps (GPU busy throughout)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    input_bytes = x.numel() * x.element_size() + y.numel() * y.element_size()
    l2_flush = input_bytes < L2_BYTES
    if not l2_flush:  # inputs larger than L2: back-to-back steps, one event pair
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / args.steps
    else:  # inputs fit in L2: write a 2x-L2 buffer between steps, outside the timed region
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        total = 0.0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            total += e0.elapsed_time(e1)
        ms = total / args.steps
    clocks.__exit__()
    launches = ctx.launches - launches0
    # per-kernel times: the same K steps again, untimed, with an event pair around every launch (the events
    # would add their own gaps to the timed region above)
    # The fp64 path's timed steps run K1Q's cut beside the Gram (one launch region); each kernel's own duration
    # (the rooflines) comes from this pass in the serial schedule (CVG_I8_OVERLAP=0: every kernel alone on the
    # GPU), and a second pass in the step's own schedule times the shared region.
    def kernel_pass(overlap):
        prev = os.environ.get("CVG_I8_OVERLAP")
        if overlap is not None:
            os.environ["CVG_I8_OVERLAP"] = overlap
        L.lib().cvg_context_enable_timing(ctx.handle, 1)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize(dev)
        t, c = np.zeros(6), np.zeros(6, np.int64)
        L.lib().cvg_context_kernel_times(ctx.handle, t.ctypes.data, c.ctypes.data)
        L.lib().cvg_context_enable_timing(ctx.handle, 0)
        if overlap is not None:
            if prev is None:
                del os.environ["CVG_I8_OVERLAP"]
            else:
                os.environ["CVG_I8_OVERLAP"] = prev
        return t, c

    kms, kcnt = kernel_pass("0")
    kms_step, _ = kernel_pass(None) if x.dtype == torch.float64 else (kms, None)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        kt = torch.tensor(np.stack([kms, kms_step]), device=dev)
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)
        kms, kms_step = kt.cpu().numpy()
    value = flops / (ms * 1e-3) / 1e9
    x_elt = x.element_size()

    # ---- e2e through the reference-facing C ABI with pinned host buffers (N=1)
    e2e = None
    sharded_e2e = args.e2e_path == "sharded" or (args.e2e_path == "auto" and world > 1)
    if not args.no_e2e and not sharded_e2e:
        hx = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        hy = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
        hl = torch.empty(labels.shape, dtype=torch.int32, pin_memory=True)
        hx.copy_(x)
        hy.copy_(y)
        hl.copy_(labels)
        del x, y
        plan = None
        out = None
        torch.cuda.empty_cache()
        nc = len(masks)
        hxtx = torch.empty((nc, p, k, k), dtype=torch.float64, pin_memory=True)
        hxty = torch.empty((nc, p, k, m), dtype=torch.float64, pin_memory=True)
        hv = {nm: torch.empty((nc, p, d), dtype=torch.float64, pin_memory=True)
              for nm, d in (("mx", k), ("my", m), ("sx", k), ("sy", m))}
        hnt = np.empty(p, np.int64)
        hnv = np.empty(p, np.int64)
        cm = np.array(masks, np.uint32)
        dtype_code = L.DTYPE_F32 if hx.dtype == torch.float32 else L.DTYPE_F64
        ctx.set_stream(None)

        def e2e_step():
            buf = L.err_buf()
            rc = L.lib().cvg_run_all_folds(ctx.handle, dtype_code, hx.data_ptr(), hy.data_ptr(), n, k, m,
                                           hl.data_ptr(), n, p, cm.ctypes.data, nc, hxtx.data_ptr(), hxty.data_ptr(),
                                           hv["mx"].data_ptr(), hv["my"].data_ptr(), hv["sx"].data_ptr(),
                                           hv["sy"].data_ptr(), hnt.ctypes.data, hnv.ctypes.data, buf, len(buf))
            if rc:
                raise RuntimeError(buf.value.decode())

        e2e_step()
        e_steps = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
        elt = hx.element_size()
        h2d = n * k * elt + n * m * elt + n * 4
        d2h = nc * (p * k * k * 8 + p * k * m * 8 + p * (2 * k + 2 * m) * 8)
        e2e = {"value": round(flops / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "ms_per_step": round(e2e_ms, 3),
               "steps": e_steps, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "path": "cvg_run_all_folds (C ABI) from pinned host buffers, wall clock around the synchronous call"}

    elif not args.no_e2e:
        # N GPUs from HOST memory: each rank holds its row shard (pinned) and all labels,
        # copies the shard over its own PCIe link, rows go to their fold's owner over NVLink,
        # then the same fold-range run; the owned folds' outputs come back to host.
        lo, hi = P.shard_rows(n, rank, world)
        hx = torch.empty((hi - lo, k), dtype=x.dtype, pin_memory=True)
        hy = torch.empty((hi - lo, m), dtype=y.dtype, pin_memory=True)
        hl = torch.empty(labels.shape, dtype=torch.int32, pin_memory=True)
        hx.copy_(x[lo:hi])
        hy.copy_(y[lo:hi])
        hl.copy_(labels)
        elt = x.element_size()
        del x, y
        plan = None
        out = mine = gathered = None
        torch.cuda.empty_cache()
        e_plan = P.DevicePlan(n, k, m, p, dtype="f32" if elt == 4 else "f64", ctx=ctx, rank=rank, world=world)
        host_out = None

        def e2e_step():
            nonlocal host_out
            _, host_out = P.run_all_folds_sharded(hx, hy, hl, p, masks, n, plan=e_plan, device=dev,
                                                  out_host=host_out)

        e2e_step()
        e_steps = max(2, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        torch.cuda.synchronize(dev)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        nc = len(masks)
        h2d = n * k * elt + n * m * elt + world * n * 4
        d2h = nc * (p * k * k * 8 + p * k * m * 8) + p * (2 * k + 2 * m) * 8
        e2e = {"value": round(flops / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "ms_per_step": round(e2e_ms, 3),
               "steps": e_steps, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "path": "plan.run_all_folds_sharded: per-rank pinned host row shard -> own PCIe H2D -> NCCL "
                       "all-to-all of rows to their fold's owner (all-gather when P < N) -> fold-range run -> "
                       "owned folds D2H; wall clock, max over ranks; bytes are whole-job totals"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    line = {
        "metric": "all_fold_cv_gram_gflops", "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if x_dtype_is_f64(cid) else "f32",
        "data": data_note, "config": bench_config(cid),
        "l2": (f"inputs {input_bytes / 1e9:.1f} GB > 126 MB L2: no flush needed" if not l2_flush else
               f"inputs {input_bytes / 1e6:.1f} MB < 126 MB L2: L2 flushed (252 MB write) before each timed "
               f"step, steps timed individually"),
    }
    line.update(rooflines(cid, n, k, m, p, masks, world, flops, kms, kcnt, args.steps, x_elt))
    if kms_step is not kms and kms_step[1] < 0.5 * kms[1]:  # the step's schedule merged K1Q into the Gram region
        region = float(kms_step[2]) / args.steps
        line["schedule"] = {
            "cut_beside_gram_ms": round(region, 4),
            "serial_cut_plus_gram_ms": round(float(kms[1] + kms[2]) / args.steps - float(kms_step[1]) / args.steps, 4),
            "note": "timed steps: the int8 digit cut (direct-store K1Q, one CTA per SM) runs beside the lean Gram "
                    "(CVG_I8_OVERLAP=0 restores K1Q -> Gram); roofline / hbm_rooflines / kernels_ms_per_step time "
                    "each kernel alone (serial-schedule pass), cut_beside_gram_ms is the shared region of the "
                    "step's own schedule, serial_cut_plus_gram_ms the same two kernels back to back"}
        line["roofline"]["launch_ms_in_step"] = round(region, 4)
    line["gpu_launches"] = int(launches)
    line["clocks"] = clocks.summary()
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        w = host if host is not None and host.n <= CPU_SAMPLE_ROWS else cpu_sample(cid, CPU_SAMPLE_ROWS)
        times, cores = time_r64(w, 1, 3)
        t = min(times)
        t_np = time_numpy(w, 2)
        line["cpu_baseline"] = {"value": round(w.flops / t / 1e9, 3), "unit": "GFLOP/s", "cores": cores, "kind": "port",
                                "sample": r64_desc(w, cores, len(times), "min"), "host": host_cpu(),
                                "numpy_openblas": {"value": round(w.flops / t_np / 1e9, 3), "unit": "GFLOP/s",
                                                   "cores": cores, "sample": "the same workload through "
                                                   "oracle/numpy_alg7.py (fast.hpp Algorithm 7 with numpy's fp64 "
                                                   "GEMM, OpenBLAS on all host threads), min of 2 runs"}}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def rooflines(cid, n, k, m, p, masks, world, flops, kms, kcnt, steps, x_elt):
    """roofline (the Gram) and the HBM rooflines of the other kernels, from the per-class CUDA-event times."""
    from paper_2401_13185_b200.plan import executed_gram_flops
    from paper_2401_13185_b200.plan import fp64_kind as executed_fp64_kind
    from paper_2401_13185_b200.plan import i8_pairs, i8_slices

    gram_ms = kms[2] / max(kcnt[2], 1) if world == 1 else kms[2] / steps
    gram_flops_per_launch = flops / max(world, 1)
    algorithmic_tf = gram_flops_per_launch / (gram_ms * 1e-3) / 1e12
    f32 = not x_dtype_is_f64(cid)
    executed = executed_gram_flops(n, k, m, p, f32) / max(world, 1) / (gram_ms * 1e-3) / 1e12
    tf32_kind = os.environ.get("CVG_FP32_KIND") == "tf32"
    i8_kind = not f32 and executed_fp64_kind() == "i8"
    if i8_kind:
        s_ = i8_slices()
        gram_kernel = (f"gram_i8_kernel<{s_}, 64> (tcgen05.mma kind::i8: exact base-256 int8 digit slices, "
                       f"{i8_pairs(s_)} slice-pair products into int32 TMEM, exact fp64 drain)")
        peak, unit = INT8_PEAK_TOPS, "TOPS (int8)"
        peak_source = (INT8_PEAK_SOURCE + "; achieved = int8 tensor ops the kernel issues per second (128x64 tiles "
                       "covering the upper 64x64 tiles x slice pairs); its fp64-equivalent rate is fp64_equivalent")
        achieved = executed
    elif f32 and tf32_kind:
        gram_kernel = "gram_tf32_kernel (tcgen05.mma kind::tf32, 3xTF32, TMEM accumulators; CVG_FP32_KIND=tf32)"
        peak, unit, achieved = TF32_PEAK_TFLOPS, "TFLOP/s", executed
        peak_source = "measured cuBLAS TF32 GEMM 8192^3 sustained (profiles/r01_fp64_peaks.txt); executed TF32 flops"
    elif f32:
        gram_kernel = ("gram_f16s_kernel (tcgen05.mma kind::f16: power-of-two scaled fp16 hi+lo split, "
                       "3 products, TMEM accumulators, exact unscale into fp64)")
        peak, unit, achieved = peaks().get("bf16_tflops_sustained", 1385.9), "TFLOP/s", executed
        peak_source = ("MEASURED_PEAKS.json bf16_tflops_sustained (kind::f16 runs fp16 and bf16 at one rate); "
                       "achieved = executed fp16 tensor flops (3 products per entry)")
    else:
        gram_kernel = "gram_f64_kernel (DMMA.8x8x4)"
        peak, unit, achieved = FP64_DMMA_PEAK_TFLOPS, "TFLOP/s", algorithmic_tf
        peak_source = "measured DMMA issue-loop peak (profiles/r01_fp64_peaks.txt); algorithmic flops 2NK(K+M)"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_gram_ncu.json")
    if os.path.exists(tpath) and cid == 1 and i8_kind:
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    kernel_names = ["bucket", "reorder", "gram", "tree_sum", "fold_stats", "products"]
    per_kernel = {nm: round(float(kms[i]) / steps, 4) for i, nm in enumerate(kernel_names)}
    hbm = peaks().get("hbm_gbs", 6550.7)
    tile = 128 if f32 and not i8_kind else 64
    kp = -(-(k + m + 1) // tile) * tile
    if i8_kind:  # segment maxima over a 1/16 row sample + K1Q (read x | y, write S int8 digit slices)
        sample = max(1, int(os.environ.get("CVG_I8_SAMPLE", "16") or 16))
        reorder_bytes = int(n * (k + m) * x_elt * (1 + 1 / sample)) + n * kp * i8_slices()
    else:
        z_elem = 4 if (f32 and not tf32_kind) else 8  # Z: fp64 | fp16 hi + lo | tf32 hi + lo
        reorder_bytes = n * (k + m) * x_elt + n * kp * z_elem
    # epilogue, algorithmic minimum: each fold partial's upper triangle + its XᵀY block read once, every
    # configuration's outputs written once (statistics vectors are < 0.1% and left out)
    nf = p / max(world, 1)
    epi_bytes = int(8 * nf * (k * (k + 1) / 2 + k * m) + 8 * len(masks) * nf * k * (k + m))
    epi_ms = (kms[4] + kms[5]) / steps
    return {
        "roofline": {"bound": "tensor", "kernel": gram_kernel, "achieved": round(achieved, 3), "peak": peak,
                     "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_source, "launch_ms": round(gram_ms, 4),
                     "algorithmic_flops_per_launch": gram_flops_per_launch,
                     "note": "algorithmic flops = 2NK(K+M) (BASELINE metric); traffic = ncu dram bytes per launch "
                             "(profiles/r02_gram_ncu.json) for configs[1]"},
        "fp64_equivalent": {"gram_tflops": round(algorithmic_tf, 3),
                            "step_tflops": round(flops / max(world, 1) / (sum(kms) / steps * 1e-3) / 1e12, 3)
                            if sum(kms) else None,
                            "peak_tflops": FP64_DMMA_PEAK_TFLOPS, "gram_frac": round(algorithmic_tf / FP64_DMMA_PEAK_TFLOPS, 3),
                            "peak_source": "measured FP64 DMMA issue loop (profiles/r01_fp64_peaks.txt; cuBLAS "
                                           "DGEMM 35.4)",
                            "note": "BASELINE's '% of FP64 roofline': algorithmic 2NK(K+M) flops per second of the "
                                    "Gram (and of the whole device step) against the FP64 tensor peak"},
        "kernels_ms_per_step": per_kernel,
        "hbm_rooflines": {
            "reorder": {"bytes": reorder_bytes, "ms": round(kms[1] / steps, 4),
                        "achieved_gbs": round(reorder_bytes / (kms[1] / steps * 1e-3) / 1e9, 1) if kms[1] else None,
                        "peak_gbs": hbm, "frac": round(reorder_bytes / (kms[1] / steps * 1e-3) / 1e9 / hbm, 3)
                        if kms[1] else None},
            "epilogue": {"bytes": epi_bytes, "ms": round(epi_ms, 4),
                         "achieved_gbs": round(epi_bytes / (epi_ms * 1e-3) / 1e9, 1) if epi_ms else None,
                         "peak_gbs": hbm, "frac": round(epi_bytes / (epi_ms * 1e-3) / 1e9 / hbm, 3) if epi_ms else None,
                         "bytes_note": "algorithmic minimum: P fold partials' upper triangle + XᵀY block read once, "
                                       "n_cfg x P x K(K+M) outputs written once"}},
    }


def x_dtype_is_f64(cid):
    import workloads

    return workloads.DTYPES[cid] == np.float64


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
