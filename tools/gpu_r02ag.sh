#!/bin/bash
# K3a probes on C4: 1 = count pre-test candidates, 2 = no exact tests, 3 = no epilogue math
mkdir -p gpurun_out
P=${TAG:-r02ag}
for V in default hp1 hp2 hp3; do
  if [ $V = default ]; then unset SSJB_LIB; else export SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_$V.so; fi
  for K in 4096 2048; do
    echo "== $V K=$K" >> gpurun_out/${P}_heavy.jsonl
    SSJB_HEAD_K=$K timeout 300 python tools/heavy_phases.py C4 2>&1 | grep -v "^head probe" | cut -c1-700 >> gpurun_out/${P}_heavy.jsonl
    SSJB_HEAD_K=$K timeout 300 python tools/heavy_phases.py C4 2>&1 | grep "^head probe" | tail -3 >> gpurun_out/${P}_heavy.jsonl
  done
done
