#!/bin/bash
# Profiling pass: K2 pipeline trace on C4, ncu --set full of the head kernel,
# then compute-sanitizer (memcheck / racecheck / synccheck) over the fixture workload.
mkdir -p gpurun_out
P=${TAG:-r02g}
rm -f gpurun_out/tc_trace.txt
SSJB_TC_DEBUG=2 timeout 300 python tools/heavy_phases.py C4 > gpurun_out/${P}_c4_trace_run.jsonl 2>&1
python tools/trace_summary.py gpurun_out/tc_trace.txt > gpurun_out/${P}_c4_trace_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_overlap" -c 1 \
  -o gpurun_out/${P}_head python tools/heavy_phases.py C4 > gpurun_out/${P}_ncu_head.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py > gpurun_out/${P}_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/${P}_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize.py tcm l2gemm head > gpurun_out/${P}_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/${P}_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize.py tcm l2gemm head > gpurun_out/${P}_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/${P}_synccheck.log
