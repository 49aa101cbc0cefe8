#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02bl}
timeout 1200 python -m pytest tests/test_gpu_prefix.py -x -q -k full_size > gpurun_out/${P}_pytest_prefix_full.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_prefix_full.log
