"""Aggregate ncu per-SASS warp-stall samples by CUDA source line.

usage: ncu_lines.py <sass.csv from `ncu -i X --page source --csv --print-source sass`>
                    <nvdisasm --print-line-info listing of the same kernel> [top]
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]  # one kernel's SASS rows (headers skipped)
base = int(data[0][0], 16)
line_of = {}
cur = None
for l in open(sys.argv[2]):
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m and '//##' in l:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
col = hdr.index('Warp Stall Sampling (All Samples)')
ex = hdr.index('Instructions Executed')
agg = defaultdict(lambda: [0, 0])
for r in data:
    off = int(r[0], 16) - base
    ln = line_of.get(off, ('?', -1))
    agg[ln][0] += int(r[col] or 0)
    agg[ln][1] += int(r[ex] or 0)
tot = sum(v[0] for v in agg.values())
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
srcs = {}
for (fn, ln), (smp, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    text = ''
    for d in ('paper_1609_07228_b200/csrc/',):
        try:
            text = srcs.setdefault(fn, open(d + fn).read().split('\n'))[ln - 1].strip()[:70]
        except (OSError, IndexError):
            pass
    print(f"{fn[:14]:14s} {ln:5d}  samples {smp:8d} ({100 * smp / tot:5.1f}%)  inst {n:12d}  {text}")
