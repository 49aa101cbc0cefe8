#!/bin/bash
# Pipeline probes of the tcgen05 filter: 1-D bulk-copy throughput per SM, and
# CTA-0 event traces of the C2 tau=0.7 join with and without the epilogue.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk_probe tools/bulk_probe.cu && /tmp/bulk_probe > gpurun_out/bulk_probe.txt 2>&1
rm -f gpurun_out/tc_trace.txt
python - <<'PY' > gpurun_out/trace_runs.txt 2>&1
import os, sys
sys.path.insert(0, ".")
import paper_1711_07295_b200 as pkg
from paper_1711_07295_b200 import datasets as D, ssjoin as S
lib = pkg.load_library()
coll = D.c2(lib)
S.pin_device(coll, 0)
for dbg in ("0", "1", "2", "3"):
    os.environ["SSJB_TC_DEBUG"] = dbg
    for rep in range(3):
        r = S.join(coll, D.c2_options(lib, (7, 10)))
    print("debug", dbg, "filter_ms", r.extra["ms_filter"], flush=True)
PY
