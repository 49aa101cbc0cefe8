#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02bi}
for k in 1 2; do
SSJB_HOST_TIMING=2 SSJB_BENCH_DEBUG=1 SSJB_BENCH_NO_CLOCKS=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/${P}_$k.json 2> gpurun_out/${P}_$k.err
done
