#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02k}
for V in default sets1; do
  if [ $V = default ]; then unset SSJB_LIB; else export SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_$V.so; fi
  echo "== $V" >> gpurun_out/${P}_variants.txt
  timeout 300 python tools/heavy_phases.py C4 C5 2>&1 | cut -c1-460 >> gpurun_out/${P}_variants.txt
done
unset SSJB_LIB
rm -f gpurun_out/tc_trace.txt
SSJB_TC_DEBUG=2 timeout 300 python tools/heavy_phases.py C4 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/tc_trace.txt > gpurun_out/${P}_c4_trace_summary.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join or overflow or random or level3 or shard" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 900 python -m pytest tests/test_naive_rs.py -x -q -s > gpurun_out/${P}_rs_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_rs_tests.log
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "C4" > gpurun_out/${P}_heavy.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy.log
