#!/bin/bash
# Prefix-filter engine on the GPU: fixtures vs the reference, live-reference
# parity, a memcheck pass over a fixture subset, and joins on C1-C3.
mkdir -p gpurun_out
P=${TAG:-r02ap}
timeout 900 python -m pytest tests/test_gpu_prefix.py -x -q > gpurun_out/${P}_pytest_prefix.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_prefix.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k prefix_filter > gpurun_out/${P}_pytest_prefix_live.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_prefix_live.log
timeout 900 python tools/prefix_phases.py c1 c2 c3 > gpurun_out/${P}_prefix_phases.jsonl 2> gpurun_out/${P}_prefix_phases.err; echo "rc=$?" >> gpurun_out/${P}_prefix_phases.err
timeout 300 python tools/heavy_phases.py C3 > gpurun_out/${P}_heavy_c3.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_heavy_c3.log
