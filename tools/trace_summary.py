#!/usr/bin/env python3
"""Summarise gpurun_out/tc_trace.txt (CTA-0 event timestamps of the tcgen05
filter, SSJB_TC_DEBUG=2): per-tile MMA issue interval, producer lead, epilogue
duration per warp."""
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tc_trace.txt"
for bi, b in enumerate(x for x in open(path).read().split("---\n") if x.strip()):
    a = np.array([[int(x) for x in line.split()] for line in b.strip().split("\n")], dtype=np.float64)
    v = a[(a[:, 1] > 0) & (a[:, 2] > 0)]
    if len(v) < 10:
        continue
    t0 = v[0, 1]
    prod, mb, ma = v[:, 1] - t0, v[:, 2] - t0, v[:, 3] - t0
    es, ee = v[:, 4:20] - t0, v[:, 20:36] - t0
    d = np.diff(ma)
    print(f"run {bi}: tiles {len(v)}  mma interval median {np.median(d):.0f} mean {d.mean():.0f} | "
          f"mma waits on acc_empty {np.median(ma - mb):.0f} | tma latency {np.median(mb - prod):.0f} | "
          f"epi per-warp {np.median(ee - es):.0f} span {np.median(ee.max(1) - es.min(1)):.0f} | "
          f"epi start - mma issue {np.median(es.min(1) - ma):.0f}")
