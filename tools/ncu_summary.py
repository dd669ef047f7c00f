"""Summarise an ncu --set full report (.ncu-rep) into the per-kernel JSON kept under profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep "source description" > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]


def main():
    rep, source = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for r in data:
        rec = {"kernel": r[head.index("Kernel Name")][:90]}
        for m in METRICS:
            if m in head:
                i = head.index(m)
                rec[m] = r[i] + (f" {units[i]}" if units[i] else "")
        kernels.append(rec)
    print(json.dumps({"source": source, "kernels": kernels}, indent=1))


if __name__ == "__main__":
    main()
