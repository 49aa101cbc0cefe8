#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02bg}
for k in 1 2 3; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/${P}_bench_$k.json 2> gpurun_out/${P}_bench_$k.err
done
