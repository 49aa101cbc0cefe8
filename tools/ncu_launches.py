#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total/mean device time and share of the total."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki]][0] += 1
            agg[r[ki]][1] += float(r[vi].replace(",", ""))  # ns
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total ms | mean us | share |\n|---|---|---|---|---|")
    for k, (c, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:70]}` | {c} | {ns / 1e6:.3f} | {ns / c / 1e3:.1f} | {100 * ns / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
