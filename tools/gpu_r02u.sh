#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02u}
timeout 300 python tools/k1_probe.py C4 > gpurun_out/${P}_k1.txt 2>&1
SSJB_FLAT_MIN_MEAN=1000000 timeout 300 python tools/k1_probe.py C4 > gpurun_out/${P}_k1_sub.txt 2>&1
timeout 300 python tools/k1_probe.py C2 >> gpurun_out/${P}_k1.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "not sharded" > gpurun_out/${P}_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy_tests.log
