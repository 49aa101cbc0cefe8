#!/bin/bash
# A/B: chunked (8 tokens per round) thread-per-pair verify vs chunk 0 (step merge), 4, 16
mkdir -p gpurun_out
P=${TAG:-r02ad}
for V in default vq0 vq4 vq16 default vq0; do
  if [ $V = default ]; then unset SSJB_LIB; else export SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_$V.so; fi
  echo "== $V" >> gpurun_out/${P}_heavy.jsonl
  timeout 300 python tools/heavy_phases.py C3 C4 2>&1 | cut -c1-600 >> gpurun_out/${P}_heavy.jsonl
done
unset SSJB_LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 900 python -m pytest tests/test_gpu_heavy.py -x -q -s > gpurun_out/${P}_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy_tests.log
