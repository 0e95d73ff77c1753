"""Summarise an .ncu-rep: key SOL / memory / warp-state metrics per kernel launch."""
import csv
import io
import subprocess
import sys

KEEP = {
    "GPU Speed Of Light Throughput": ["Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
                                      "L2 Cache Throughput", "Compute (SM) Throughput"],
    "Memory Workload Analysis": ["Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth"],
    "Compute Workload Analysis": ["Issue Slots Busy", "Executed Ipc Active"],
    "Occupancy": ["Achieved Occupancy", "Theoretical Occupancy"],
    "Warp State Statistics": ["Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp"],
}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    cur = None
    for r in rows[1:]:
        kid = (r[col["ID"]], r[col["Kernel Name"]].split("(")[0].split("::")[-1])
        if kid != cur:
            cur = kid
            print(f"=== [{kid[0]}] {kid[1]}")
        sec, name = r[col["Section Name"]], r[col["Metric Name"]]
        if sec in KEEP and name in KEEP[sec]:
            print(f"   {sec[:24]:24s} {name:38s} {r[col['Metric Value']]:>14s} {r[col['Metric Unit']]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    names = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
             "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]
    units = rr[1]
    for r in rr[2:]:
        print(f"--- raw [{r[0]}] {r[h.index('Kernel Name')].split('(')[0].split('::')[-1]}")
        for n in names:
            if n in h:
                i = h.index(n)
                print(f"   {n:80s} {r[i]:>16s} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
