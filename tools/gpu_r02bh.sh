#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02bh}
for k in 1 2 3; do
SSJB_BENCH_DEBUG=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/${P}_clk_$k.json 2> gpurun_out/${P}_clk_$k.err
SSJB_BENCH_DEBUG=1 SSJB_BENCH_NO_CLOCKS=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/${P}_noclk_$k.json 2> gpurun_out/${P}_noclk_$k.err
done
