#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases128.jsonl 2>&1
SSJB_HOST_TIMING=1 timeout 300 python tools/host_overhead.py pinned > gpurun_out/ho_pinned.json 2> gpurun_out/ho_pinned.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
