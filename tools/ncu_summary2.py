"""Writes a text summary of every launch in an .ncu-rep (--set full): duration,
SOL, IPC, occupancy, DRAM bytes, tensor-pipe activity, top stall reasons.
python tools/ncu_summary2.py report.ncu-rep > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size"]
stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_") or
         (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"))]
print(f"# {rep}")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print(f"\n## {r[hdr.index('ID')]} {name[:110]}")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:70s} {r[i]:>16s} {units[i]}")
    st = []
    for h in stall:
        try:
            st.append((float(r[hdr.index(h)].replace(",", "")), h))
        except ValueError:
            pass
    tot = sum(v for v, _ in st) or 1.0
    for v, h in sorted(st, reverse=True)[:8]:
        print(f"  stall {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):60s} {100 * v / tot:6.1f}%")
