#!/bin/bash
# Round-2 evidence pass: GPU tests, smoke, bench (both arms, C4 headline),
# launch list of the bench, ncu --set full of the C4 join's kernels.
mkdir -p gpurun_out
P=${TAG:-r02d}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_gpu.txt 2>&1
lscpu > gpurun_out/${P}_lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/${P}_bench_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"filter_tc_kernel|head_overlap|verify_pairs|build_sketches" -c 7 \
  -o gpurun_out/${P}_c4_kernels python tools/heavy_phases.py C4 > gpurun_out/${P}_ncu_full.log 2>&1
ls -la gpurun_out | tail -30
