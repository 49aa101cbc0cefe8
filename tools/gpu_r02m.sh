#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02m}
timeout 300 python tools/heavy_phases.py C4 C3 > gpurun_out/${P}_heavy_phases.jsonl 2>&1
rm -f gpurun_out/tc_trace.txt
SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_trace.so SSJB_TC_DEBUG=2 timeout 300 python tools/heavy_phases.py C4 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/tc_trace.txt > gpurun_out/${P}_c4_trace_summary.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_naive_rs.py tests/test_delivery.py -x -q > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s > gpurun_out/${P}_heavy.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy.log
