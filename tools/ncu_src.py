"""Per-CUDA-line warp-stall samples and executed instructions of one kernel launch
in an .ncu-rep (build with -lineinfo):
    python tools/ncu_src.py report.ncu-rep <kernel-regex> [launch-skip] [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r[0].isdigit() and r[hdr["Address"]] == "-":
        smp = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        ins = int(r[hdr["Instructions Executed"]] or 0)
        if smp or ins:
            rows.append((smp, ins, fname, int(r[0]), r[1].strip()[:80]))
tot_s = sum(r[0] for r in rows) or 1
tot_i = sum(r[1] for r in rows) or 1
print(f"{tot_s} samples, {tot_i} warp instructions")
for smp, ins, fn, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{fn[:12]:12s} {ln:5d} {100 * smp / tot_s:5.1f}% smp {100 * ins / tot_i:5.1f}% ins  {src}")
