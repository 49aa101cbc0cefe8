#!/bin/bash
# Prefix-filter engine: tests, joins on C1-C3, ncu of the encounter kernel on C3.
mkdir -p gpurun_out
P=${TAG:-r02ar}
timeout 900 python -m pytest tests/test_gpu_prefix.py -x -q > gpurun_out/${P}_pytest_prefix.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_prefix.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k prefix_filter > gpurun_out/${P}_pytest_prefix_live.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_prefix_live.log
timeout 900 python tools/prefix_phases.py c1 c2 c3 > gpurun_out/${P}_prefix_phases.jsonl 2> gpurun_out/${P}_prefix_phases.err; echo "rc=$?" >> gpurun_out/${P}_prefix_phases.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefix_encounters|adapt_tally" -c 2 \
  -o gpurun_out/${P}_c3_prefix python tools/prefix_phases.py c3 --algo 2 --bitmap f3 --reps 1 > gpurun_out/${P}_ncu_c3.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_ncu_c3.log
