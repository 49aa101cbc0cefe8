#!/bin/bash
# K3a head width sweep on C4: head kernel vs verify time
mkdir -p gpurun_out
P=${TAG:-r02af}
for K in 2048 3072 4096 2560 3584; do
  echo "== K=$K" >> gpurun_out/${P}_heavy.jsonl
  SSJB_HEAD_K=$K timeout 300 python tools/heavy_phases.py C4 2>&1 | cut -c1-700 >> gpurun_out/${P}_heavy.jsonl
done
