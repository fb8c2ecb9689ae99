"""Summarise an ncu report (details page) into the metrics we track.

    python profiles/ncu_summary.py gpurun_out/x.ncu-rep [--all]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM",
        "Registers Per Thread", "Executed Instructions", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block",
        "Compute (SM) Throughput", "Branch Efficiency", "Local Memory Spilling Requests"]


def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ik, iname, iunit, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index(
        "Metric Value")
    res = {}
    for r in rows[1:]:
        res.setdefault(r[ik], {})[r[iname]] = (r[ival], r[iunit])
    return res


def raw(path, metrics):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    vals = {}
    for m in metrics:
        if m in hdr:
            vals[m] = [r[hdr.index(m)] for r in rows[2:]]
    return vals


if __name__ == "__main__":
    path = sys.argv[1]
    for k, d in details(path).items():
        print(k)
        for key in (d if "--all" in sys.argv else KEYS):
            if key in d:
                print(f"  {key:40s} {d[key][0]} {d[key][1]}")
    rv = raw(path, ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "gpu__time_duration.sum"])
    for m, v in rv.items():
        print(f"  {m:40s} {v}")
