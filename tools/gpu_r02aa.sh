#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02aa}
timeout 300 python tools/heavy_phases.py C4 2>&1 | cut -c1-460 > gpurun_out/${P}_heavy.jsonl
SSJB_HEAD_WARP_VERIFY=0 timeout 300 python tools/heavy_phases.py C4 2>&1 | cut -c1-460 >> gpurun_out/${P}_heavy.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"filter_tc_kernel" -c 1 \
  -o gpurun_out/${P}_k2 python tools/heavy_phases.py C4 > gpurun_out/${P}_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join or overflow" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "C4 and not sharded" > gpurun_out/${P}_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy_tests.log
