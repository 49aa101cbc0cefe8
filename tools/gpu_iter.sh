#!/bin/bash
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases128.jsonl 2>&1
SSJB_TCM=0 timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases128_1tile.jsonl 2>&1
timeout 300 python tools/c2_phases.py 64 3 > gpurun_out/phases64.jsonl 2>&1
SSJB_TCM=0 timeout 300 python tools/c2_phases.py 64 3 > gpurun_out/phases64_1tile.jsonl 2>&1
