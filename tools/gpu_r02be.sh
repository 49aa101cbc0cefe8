#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02be}
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "two_phase or streamed or head or every_golden or overflow" > gpurun_out/${P}_pytest_a.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_a.log
timeout 1500 python -m pytest tests/test_gpu_heavy.py -x -q > gpurun_out/${P}_pytest_heavy.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_heavy.log
timeout 600 python tools/c4_gaps.py > gpurun_out/${P}_c4_gaps.jsonl 2> gpurun_out/${P}_c4_gaps.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "rc=$?" >> gpurun_out/${P}_bench.err
