#!/bin/bash
# A/B: level-2 GEMM column sizes from the shared side ring (default) vs global loads
mkdir -p gpurun_out
P=${TAG:-r02ab}
for V in default noring ring4 default noring ring4; do
  if [ $V = default ]; then unset SSJB_LIB; else export SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_$V.so; fi
  echo "== $V" >> gpurun_out/${P}_heavy.jsonl
  timeout 300 python tools/heavy_phases.py C4 2>&1 | cut -c1-420 >> gpurun_out/${P}_heavy.jsonl
done
unset SSJB_LIB
#timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join or overflow or random or level3 or streamed or sketch" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
#timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "not sharded" > gpurun_out/${P}_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy_tests.log
