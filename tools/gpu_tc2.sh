#!/bin/bash
# First run of the CTA-pair filter: guarded smoke, parity, A/B phase timing.
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
if grep -q "rc=0" gpurun_out/smoke.log; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
  timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases_tc2.jsonl 2>&1
  SSJB_TC2=0 timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases_tc1.jsonl 2>&1
  SSJB_LIB=$PWD/paper_1711_07295_b200/lib/libssjoin_head.so timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases_head.jsonl 2>&1
  timeout 900 python tools/heavy_phases.py C3 C5 C4 > gpurun_out/heavy_phases.jsonl 2>&1
fi
