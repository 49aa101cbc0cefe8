#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02z}
for D in 2 3; do
  rm -f gpurun_out/tc_trace.txt
  SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_trace.so SSJB_TC_DEBUG=$D timeout 300 python tools/heavy_phases.py C4 > /dev/null 2>&1
  echo "== SSJB_TC_DEBUG=$D" >> gpurun_out/${P}_trace.txt
  python tools/trace_summary.py gpurun_out/tc_trace.txt >> gpurun_out/${P}_trace.txt 2>&1
done
