"""Aggregates an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv
import sys
from collections import defaultdict


def main(path, title=""):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    kc, mc, vc = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= vc or r[mc] != "gpu__time_duration.sum":
            continue
        name = r[kc].split("(")[0].split("::")[-1].split("<")[0] or r[kc][:40]
        v = float(r[vc].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    if title:
        print(f"# {title}")
    print(f"# total kernel time {tot:.1f} ms over {sum(v[0] for v in agg.values())} launches")
    print(f"{'kernel':40s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:40]:40s} {c:8d} {ms:10.2f} {100 * ms / tot:6.2f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
