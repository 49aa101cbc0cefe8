#!/bin/bash
# Is the K2 per-tile fixed cost the accumulator handshake's wake-up latency?
mkdir -p gpurun_out
P=${TAG:-r02o}
for V in default nosusp susp100; do
  if [ $V = default ]; then unset SSJB_LIB; else export SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_$V.so; fi
  for D in 0 1 5; do
    echo "== $V SSJB_TC_DEBUG=$D" >> gpurun_out/${P}_probes.txt
    SSJB_TC_DEBUG=$D timeout 300 python tools/heavy_phases.py C4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('filter_ms', d['ms']['filter'], 'head_ms', d['ms']['head'], 'batches', d['batches'])" >> gpurun_out/${P}_probes.txt
  done
done
