#!/bin/bash
# C5 fp4 filter tile width: N=192 (default, 2 accumulator slots) vs N=128 (3 slots)
mkdir -p gpurun_out
P=${TAG:-r02ah}
timeout 400 python tools/heavy_phases.py C5 2>&1 | cut -c1-700 >> gpurun_out/${P}_heavy.jsonl
SSJB_TC_N=128 timeout 400 python tools/heavy_phases.py C5 2>&1 | cut -c1-700 >> gpurun_out/${P}_heavy.jsonl
SSJB_TC_N=128 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
