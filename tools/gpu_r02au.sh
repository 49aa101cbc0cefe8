#!/bin/bash
# Prefix engine: full-size + delivery tests, compute-sanitizer memcheck/racecheck/synccheck.
mkdir -p gpurun_out
P=${TAG:-r02au}
timeout 900 python -m pytest tests/test_gpu_prefix.py -x -q > gpurun_out/${P}_pytest_prefix.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_prefix.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_prefix.py > gpurun_out/${P}_san_${tool}.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_san_${tool}.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch" > gpurun_out/${P}_pytest_sketch.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_sketch.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "rc=$?" >> gpurun_out/${P}_bench.err
