#!/bin/bash
# K2 claim order + head K experiments on C4, then the parity tests touching them.
mkdir -p gpurun_out
P=${TAG:-r02e}
for K in 2048 4096; do
  SSJB_HEAD_K=$K timeout 300 python tools/heavy_phases.py C4 > gpurun_out/${P}_c4_k$K.jsonl 2>&1
done
SSJB_ITEM_ORDER=0 timeout 300 python tools/heavy_phases.py C4 > gpurun_out/${P}_c4_noorder.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join or overflow or random" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "C4 and not sharded" > gpurun_out/${P}_heavy.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy.log
