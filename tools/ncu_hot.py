"""Per-kernel SASS hot spots from an .ncu-rep (needs -lineinfo builds):
python tools/ncu_hot.py report.ncu-rep <kernel-regex> [launch-skip]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
c = {h: i for i, h in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        ins.append((r[c["Source"]].strip(), int(r[c["Warp Stall Sampling (All Samples)"]] or 0),
                    int(r[c["Instructions Executed"]] or 0)))
    except ValueError:
        break
tot = sum(i[1] for i in ins) or 1
totx = sum(i[2] for i in ins) or 1
print(f"{len(ins)} SASS instructions, {tot} samples")
for k in range(0, len(ins), 32):
    blk = ins[k:k + 32]
    s = sum(b[1] for b in blk)
    x = sum(b[2] for b in blk)
    if s / tot > 0.03:
        ops = collections.Counter((b[0].split()[1] if b[0].startswith("@") else b[0].split()[0]).split(".")[0]
                                  for b in blk)
        print(f"{k:5d} {s / tot * 100:5.1f}% samples {x / totx * 100:5.1f}% instr  {dict(ops.most_common(7))}")
