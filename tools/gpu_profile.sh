#!/bin/bash
# Evidence for profiles/: launch list of one bench run, ncu --set full of the
# C2 filter launches (8 joins), and a bench line.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -c 8 \
  -o gpurun_out/filter_tc python tools/c2_phases.py 128 1 > gpurun_out/ncu_full.log 2>&1
