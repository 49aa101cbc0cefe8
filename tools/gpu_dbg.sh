#!/bin/bash
mkdir -p gpurun_out
export SSJB_FILTER=tc SSJB_L2GEMM=0 SSJB_TC_KIND=i8 SSJB_TC2=1
timeout 300 python tools/golden_probe.py > gpurun_out/golden_probe.txt 2>&1; echo "rc=$?" >> gpurun_out/golden_probe.txt
K=$(grep -o "^FAIL [0-9]*\|^MISMATCH [0-9]*" gpurun_out/golden_probe.txt | head -1 | awk '{print $2}')
if [ -n "$K" ]; then
  timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/golden_probe.py $K > gpurun_out/sanitizer.txt 2>&1
fi
unset SSJB_FILTER SSJB_L2GEMM SSJB_TC_KIND SSJB_TC2
SSJB_TC2=0 SSJB_SURVIVOR_CAP=134217728 timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases_cap27.jsonl 2>&1
