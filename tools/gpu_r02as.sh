#!/bin/bash
# Prefix engine at 64 regs, heavy-tail sketch build, C4/C5 full pair lists, bench.
mkdir -p gpurun_out
P=${TAG:-r02as}
timeout 900 python -m pytest tests/test_gpu_prefix.py tests/test_gpu_parity.py -x -q -k "prefix or sketch" > gpurun_out/${P}_pytest_a.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_a.log
timeout 900 python tools/prefix_phases.py c1 c2 c3 > gpurun_out/${P}_prefix_phases.jsonl 2> gpurun_out/${P}_prefix_phases.err; echo "rc=$?" >> gpurun_out/${P}_prefix_phases.err
timeout 1200 python -m pytest tests/test_gpu_heavy.py -x -q -k "C4 or C5" > gpurun_out/${P}_pytest_heavy.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_heavy.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "rc=$?" >> gpurun_out/${P}_bench.err
