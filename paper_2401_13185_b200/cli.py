"""`cvgram` command line on the B200 engine (reference: proj/tools/cvgram_cli.cpp).

    python -m paper_2401_13185_b200 verify (--x X.csv --y Y.csv --partition P.txt | --random N K M P SEED) [--tol 1e-8]
    python -m paper_2401_13185_b200 run --x X.csv --y Y.csv --partition P.txt --config TOKEN --out-dir DIR [--engine fast|baseline]
    python -m paper_2401_13185_b200 bench --n N --k K --m M --p-list 10,1000 [--config TOKEN] [--reps 3] [--seed 42] --out T.csv

Exit codes (cvgram_cli.cpp:22-26): 0 ok, 2 parse/io, 3 dimension, 4 partition
invalid, 5 not scalable, 6 tolerance exceeded; 1 = the device could not run
(there is no CPU path).  `verify` runs the fast engine for all 16
configurations from ONE Gram pass and checks it against the device baseline
engine (direct per-fold recomputation).  `run` writes the reference's on-disk
format byte for byte (%.17g headerless CSV per fold + stats.csv).  The
`leakage` subcommand (the Lindgren-1994 demonstrator) is out of scope here.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import cvgram as cv

EXIT_PARSE, EXIT_DIMENSION, EXIT_PARTITION, EXIT_NOT_SCALABLE, EXIT_TOLERANCE, EXIT_DEVICE = 2, 3, 4, 5, 6, 1


class CliIOError(Exception):
    """io_error (io.hpp:19-21)."""


def read_matrix_csv(path: str) -> np.ndarray:
    """Headerless CSV, one sample per row (io.hpp:43-78): same validation."""
    try:
        f = open(path, "rb")
    except OSError:
        raise CliIOError(f"cannot open: {path}")
    rows = []
    with f:
        for raw in f.read().decode().split("\n"):
            line = raw[:-1] if raw.endswith("\r") else raw
            if not line:
                continue
            row = []
            for cell in line.split(","):
                try:
                    row.append(float(cell))
                except ValueError:
                    raise CliIOError(f"bad number '{cell}' in {path}")
            if rows and len(row) != len(rows[0]):
                raise CliIOError(f"ragged rows in {path}")
            rows.append(row)
    if not rows:
        raise CliIOError(f"empty matrix file: {path}")
    return np.array(rows, dtype=np.float64)


def write_matrix_csv(path: str, m: np.ndarray) -> None:
    """%.17g, ',' separated, '\\n' terminated (io.hpp:30-41)."""
    m = np.atleast_2d(m)
    with open(path, "w", newline="\n") as f:
        for row in m:
            f.write(",".join(cv.format_double(v) for v in row))
            f.write("\n")


def read_partition_file(path: str) -> cv.Partitioning:
    """One 1-based label per line; p = the largest label (io.hpp:81-104)."""
    try:
        text = open(path, "rb").read().decode()
    except OSError:
        raise CliIOError(f"cannot open: {path}")
    labels = []
    for raw in text.split("\n"):
        line = raw[:-1] if raw.endswith("\r") else raw
        if not line:
            continue
        try:
            labels.append(int(line))
        except ValueError:
            raise CliIOError(f"bad fold label '{line}' in {path}")
    if not labels:
        raise CliIOError(f"empty partition file: {path}")
    return cv.Partitioning(np.array(labels, np.int32), max(labels))


def load_inputs(args, allow_random: bool):
    """cvgram_cli.cpp:33-57: --random N K M P SEED draws data then labels from one stream."""
    if allow_random and args.random:
        n, k, m, p, seed = (int(v) for v in args.random)
        rng = cv.MT19937_64(seed)
        return cv.random_dataset(n, k, m, rng), cv.random_partitioning(n, p, rng)
    data = cv.DatasetPair(read_matrix_csv(args.x), read_matrix_csv(args.y))
    part = read_partition_file(args.partition)
    if part.n_rows() != data.n_rows():
        raise cv.DimensionError(f"partition file has {part.n_rows()} labels but data has {data.n_rows()} rows")
    return data, part


def cmd_verify(data, part, tol: float, ctx=None) -> int:
    err = cv.validate_partitioning(part)
    if err:
        print(f"invalid partitioning: {err}", file=sys.stderr)
        return EXIT_PARTITION
    err = cv.check_scalable(part)  # all 16 configurations run
    if err:
        print(f"partitioning not scalable: {err}", file=sys.stderr)
        return EXIT_NOT_SCALABLE
    configs = cv.enumerate_configs()
    fast = cv.run_all_folds_configs(data, part, configs, ctx=ctx)  # one Gram pass, 16 epilogues
    base = cv.baseline_fold_products_configs(data, part, configs)
    all_ok = True
    for cfg, fr, br in zip(configs, fast, base):
        worst = 0.0
        for f, b in zip(fr, br):
            worst = max(worst, cv.max_rel_diff(f.xtx_t, b.xtx_t), cv.max_rel_diff(f.xty_t, b.xty_t))
        ok = worst <= tol
        all_ok = all_ok and ok
        print(f"config {cv.config_to_string(cfg)} max_rel_diff {cv.format_double(worst)} {'ok' if ok else 'FAIL'}")
    print(("verify: all 16 configs within tolerance " if all_ok else "verify: tolerance exceeded, tol ")
          + cv.format_double(tol))
    return 0 if all_ok else EXIT_TOLERANCE


def _stats_lines(r) -> list:
    lines = [f"{r.fold_id},counts,{r.stats.n_train},{r.stats.n_val}"]
    for name, v in (("mean_x", r.stats.mean_x_t), ("mean_y", r.stats.mean_y_t), ("std_x", r.stats.std_x_t),
                    ("std_y", r.stats.std_y_t)):
        if v.size:
            lines.append(f"{r.fold_id},{name}," + ",".join(cv.format_double(x) for x in v))
    return lines


def cmd_run(data, part, cfg: cv.PreprocessConfig, engine: str, out_dir: str, ctx=None) -> int:
    """Per-fold %.17g CSVs + stats.csv (cvgram_cli.cpp:90-132).  The fast engine streams folds in batches
    (cvg_run_all_folds_stream): a writer thread formats and writes each batch while the next batch's epilogue
    and device-to-host copy run (the C call releases the GIL).  With a multi-device context (--devices) the
    folds come from one sharded run instead; the files are byte-identical either way."""
    import queue
    import threading

    err = cv.validate_partitioning(part)
    if err:
        print(f"invalid partitioning: {err}", file=sys.stderr)
        return EXIT_PARTITION
    if cfg.any_scale():
        err = cv.check_scalable(part)
        if err:
            print(f"partitioning not scalable: {err}", file=sys.stderr)
            return EXIT_NOT_SCALABLE
    os.makedirs(out_dir, exist_ok=True)
    stats = {}
    work: queue.Queue = queue.Queue(maxsize=4)
    failure = []

    def writer():
        while True:
            batch = work.get()
            if batch is None:
                return
            try:
                for r in batch:
                    tag = f"fold_{r.fold_id}"
                    write_matrix_csv(os.path.join(out_dir, tag + "_xtx.csv"), r.xtx_t)
                    write_matrix_csv(os.path.join(out_dir, tag + "_xty.csv"), r.xty_t)
                    stats[r.fold_id] = _stats_lines(r)
            except OSError as e:
                failure.append(e)

    th = threading.Thread(target=writer, daemon=True)
    th.start()
    try:
        if engine == "baseline":
            work.put(cv.baseline_fold_products(data, part, cfg))
        elif isinstance(ctx, cv.MultiContext):
            work.put(cv.run_all_folds(data, part, cfg, ctx=ctx))
        else:
            pending = []

            def take(ci, r):  # for_each_fold hands over arrays it has already copied out of the batch buffers
                pending.append(r)
                if len(pending) >= 64:
                    work.put(list(pending))
                    pending.clear()

            cv.for_each_fold(data, part, [cfg], take, batch=64, ctx=ctx)
            if pending:
                work.put(list(pending))
    finally:
        work.put(None)
        th.join()
    if failure:
        raise CliIOError(f"cannot write fold files in {out_dir}: {failure[0]}")
    stats_lines = ["fold,name,values"]
    for f in sorted(stats):
        stats_lines += stats[f]
    try:
        with open(os.path.join(out_dir, "stats.csv"), "w", newline="\n") as f:
            f.write("\n".join(stats_lines) + "\n")
    except OSError:
        raise CliIOError(f"cannot write stats.csv in {out_dir}")
    print(f"wrote {len(stats)} folds to {out_dir}")
    return 0


def _min_wall_time(reps: int, fn) -> float:
    """bench.hpp:25-35."""
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def cmd_bench(n, k, m, p_list, cfg, reps, seed, out_path) -> int:
    rng = cv.MT19937_64(seed)
    data = cv.random_dataset(n, k, m, rng)
    try:
        out = open(out_path, "w", newline="\n")
    except OSError:
        raise CliIOError(f"cannot open for writing: {out_path}")
    with out:
        out.write("engine,config,n,k,m,p,wall_time,reps\n")
        for p in p_list:
            part = cv.random_partitioning(n, p, rng)
            t_base = _min_wall_time(reps, lambda: cv.baseline_fold_products(data, part, cfg))
            t_fast = _min_wall_time(reps, lambda: cv.run_all_folds(data, part, cfg))
            for name, t in (("baseline", t_base), ("fast", t_fast)):
                out.write(f"{name},{cv.config_to_string(cfg)},{n},{k},{m},{p},{cv.format_double(t)},{reps}\n")
                print(f"{name} p={p} {cv.format_double(t)} s (min of {reps})")
    return 0


def build_parser():
    ap = argparse.ArgumentParser(prog="cvgram", description="training-partition XtX / XtY products for P-fold "
                                                            "cross-validation (B200 engine)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify", help="compare the fast engine against the baseline engine for all 16 configs")
    v.add_argument("--x")
    v.add_argument("--y")
    v.add_argument("--partition")
    v.add_argument("--random", nargs=5, metavar=("N", "K", "M", "P", "SEED"))
    v.add_argument("--tol", type=float, default=1e-8)
    v.add_argument("--threads", type=int, default=1)
    v.add_argument("--devices", default=None, help="comma-separated CUDA devices for the fast engine's run "
                                                    "(cvg_context_create_multi; results are identical)")
    r = sub.add_parser("run", help="write per-fold products and statistics to disk")
    r.add_argument("--x", required=True)
    r.add_argument("--y", required=True)
    r.add_argument("--partition", required=True)
    r.add_argument("--config", default="none")
    r.add_argument("--engine", default="fast", choices=["fast", "baseline"])
    r.add_argument("--out-dir", required=True)
    r.add_argument("--threads", type=int, default=1)
    r.add_argument("--devices", default=None)
    b = sub.add_parser("bench", help="time both engines over a sweep of fold counts")
    b.add_argument("--n", type=int, required=True)
    b.add_argument("--k", type=int, required=True)
    b.add_argument("--m", type=int, required=True)
    b.add_argument("--p-list", required=True)
    b.add_argument("--config", default="none")
    b.add_argument("--reps", type=int, default=3)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--out", required=True)
    b.add_argument("--threads", type=int, default=1)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else EXIT_PARSE
    if getattr(args, "threads", 1) < 1:
        print("--threads must be at least 1", file=sys.stderr)
        return EXIT_PARSE
    try:
        ctx = None
        if getattr(args, "devices", None):
            try:
                devs = [int(t) for t in args.devices.split(",") if t != ""]
            except ValueError:
                print(f"bad --devices list: {args.devices}", file=sys.stderr)
                return EXIT_PARSE
            ctx = cv.MultiContext(devs)
        if args.cmd == "verify":
            if not args.random and not (args.x and args.y and args.partition):
                print("verify needs --x/--y/--partition or --random", file=sys.stderr)
                return EXIT_PARSE
            data, part = load_inputs(args, allow_random=True)
            return cmd_verify(data, part, args.tol, ctx)
        if args.cmd == "run":
            cfg = cv.parse_config(args.config)
            data, part = load_inputs(args, allow_random=False)
            return cmd_run(data, part, cfg, args.engine, args.out_dir, ctx)
        if args.cmd == "bench":
            if not 3 <= args.reps <= 1000:
                print("--reps must be in [3, 1000]", file=sys.stderr)
                return EXIT_PARSE
            p_list = [int(t) for t in args.p_list.split(",") if t]
            for p in p_list:
                if p < 2 or p > args.n:
                    raise cv.PartitionError(f"fold count {p} outside {{2..N}}")
            return cmd_bench(args.n, args.k, args.m, p_list, cv.parse_config(args.config), args.reps, args.seed,
                             args.out)
    except (CliIOError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PARSE
    except cv.ScalabilityError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NOT_SCALABLE
    except cv.PartitionError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PARTITION
    except cv.DimensionError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_DIMENSION
    except cv.DeviceError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_DEVICE
    return EXIT_PARSE


if __name__ == "__main__":
    sys.exit(main())
