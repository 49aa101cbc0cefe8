#!/bin/bash
# Full GPU suite + smoke + bench at HEAD (three-tier sketch build, prefix engine).
mkdir -p gpurun_out
P=${TAG:-r02at}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch" > gpurun_out/${P}_pytest_sketch.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_sketch.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "rc=$?" >> gpurun_out/${P}_bench.err
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
