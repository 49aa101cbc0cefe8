#!/bin/bash
mkdir -p gpurun_out
for cfg in "SSJB_L2GEMM=1" "SSJB_L2GEMM=0" "SSJB_TC_N=128"; do
  env $cfg timeout 300 python tools/c2_phases.py 128 2 > gpurun_out/var.jsonl 2>&1
  python -c "
import json
rows=[json.loads(l) for l in open('gpurun_out/var.jsonl') if l.startswith('{')]
print('$cfg', [(r['tau'], r['ms']['filter'], r['ms']['verify'], r['ms']['rescan'], r['kernel']) for r in rows])"
done > gpurun_out/l2_sweep.txt 2>&1
