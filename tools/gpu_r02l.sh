#!/bin/bash
# K2 (level-2 GEMM) pipeline probes on C4: which stage paces the tile interval.
mkdir -p gpurun_out
P=${TAG:-r02l}
for D in 0 1 4 5 8 9 13; do
  echo "== SSJB_TC_DEBUG=$D" >> gpurun_out/${P}_probes.txt
  SSJB_TC_DEBUG=$D SSJB_HEAD=0 timeout 300 python tools/heavy_phases.py C4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('filter_ms', d['ms']['filter'], 'batches', d['batches'])" >> gpurun_out/${P}_probes.txt
done
