#!/bin/bash
# Final evidence at HEAD (two-phase streamed ingest): GPU tests, smoke, bench
# both arms, launch list, ncu --set full of C4's K2 / K3a / K3.
mkdir -p gpurun_out
P=${TAG:-r02bf}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
timeout 900 python tools/prefix_phases.py c1 c2 c3 > gpurun_out/${P}_prefix_phases.jsonl 2> gpurun_out/${P}_prefix_phases.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/${P}_bench_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"filter_tc_kernel|head_overlap|verify_pairs" -c 4 \
  -o gpurun_out/${P}_c4_kernels python tools/heavy_phases.py C4 > gpurun_out/${P}_ncu_c4.log 2>&1
ls -la gpurun_out | tail -20
