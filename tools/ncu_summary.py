"""Key metrics per kernel from an ncu --set full report (for profiles/)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy",
        "Eligible Warps Per Scheduler", "Grid Size", "Block Size", "L2 Hit Rate"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
       "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
       "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_not_selected"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep):
    det = list(csv.reader(run([rep, "--page", "details", "--csv"]).splitlines()))
    h = det[0]
    ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = {}
    order = []
    for r in det[1:]:
        k = r[ki].split("(")[0]
        if k not in per:
            per[k] = {}
            order.append(k)
        if r[mi] in WANT and r[mi] not in per[k]:
            per[k][r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = list(csv.reader(run([rep, "--page", "raw", "--csv", "--metrics", ",".join(RAW)]).splitlines()))
    rh = raw[0]
    for r in raw[2:]:
        k = r[rh.index("Kernel Name")].split("(")[0]
        for m in RAW:
            if m in rh:
                per.setdefault(k, {})[m.replace("smsp__pcsamp_warps_issue_stalled_", "stall_")] = r[rh.index(m)]
    for k in order:
        print(f"== {k}")
        for m, v in per[k].items():
            print(f"   {m:48s} {v}")


if __name__ == "__main__":
    main(sys.argv[1])
