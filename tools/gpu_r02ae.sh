#!/bin/bash
# verify with block-aggregated result slots: C3/C4 phases, parity + heavy tests
mkdir -p gpurun_out
P=${TAG:-r02ae}
for V in 1 2; do timeout 300 python tools/heavy_phases.py C3 C4 2>&1 | cut -c1-600 >> gpurun_out/${P}_heavy.jsonl; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join or overflow or random or level3 or streamed or sketch or naive" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 900 python -m pytest tests/test_gpu_heavy.py -x -q -s > gpurun_out/${P}_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy_tests.log
