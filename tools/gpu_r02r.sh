#!/bin/bash
# K2 probes with the head kernel on: is the level-2 GEMM filter bound by its B-tile copies?
mkdir -p gpurun_out
P=${TAG:-r02r}
for D in 0 1 8 9; do
  echo "== SSJB_TC_DEBUG=$D" >> gpurun_out/${P}_probes.txt
  SSJB_TC_DEBUG=$D timeout 300 python tools/heavy_phases.py C4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('filter_ms', d['ms']['filter'], 'batches', d['batches'], 'survivors', d['survivors_emitted'])" >> gpurun_out/${P}_probes.txt
done
