#!/bin/bash
mkdir -p gpurun_out
for cfg in "SSJB_STREAM=0" "SSJB_STREAM_CHUNKS=1" "SSJB_STREAM_CHUNKS=2" "SSJB_STREAM_CHUNKS=4" "SSJB_STREAM_CHUNKS=8" "SSJB_DELTA8=0" "SSJB_DELTA8=0 SSJB_STREAM=0"; do
  env $cfg timeout 300 python tools/host_overhead.py upload > gpurun_out/ho.json 2>&1
  python -c "
import json
d=json.load(open('gpurun_out/ho.json')); print('$cfg', d['step_ms'], [(j['tau'], j['wall'], round(j['ms']['filter'],3)) for j in d['joins']][2:4])"
done > gpurun_out/stream_sweep.txt 2>&1
