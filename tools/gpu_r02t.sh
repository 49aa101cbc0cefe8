#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02t}
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch or golden_join or streamed" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 300 python tools/heavy_phases.py C4 C2 2>&1 | cut -c1-400 > gpurun_out/${P}_heavy.jsonl
timeout 300 python tools/k1_probe.py > gpurun_out/${P}_k1.txt 2>&1
SSJB_FLAT_MIN_MEAN=1000000 timeout 300 python tools/k1_probe.py > gpurun_out/${P}_k1_sub.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "not sharded" > gpurun_out/${P}_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy_tests.log
