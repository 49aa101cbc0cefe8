#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02f}
for KIND in fp4 i8; do
  SSJB_HEAD_KIND=$KIND timeout 300 python tools/heavy_phases.py C4 > gpurun_out/${P}_c4_$KIND.jsonl 2>&1
done
SSJB_HEAD_KIND=fp4 SSJB_HEAD_K=2048 timeout 300 python tools/heavy_phases.py C4 > gpurun_out/${P}_c4_fp4_k2048.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join or overflow or random" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "not sharded" > gpurun_out/${P}_heavy.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy.log
