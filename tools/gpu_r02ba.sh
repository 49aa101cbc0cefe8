#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02ba}
timeout 600 python tools/c4_e2e_gaps.py > gpurun_out/${P}_c4_e2e_gaps.jsonl 2> gpurun_out/${P}_c4_e2e_gaps.err; echo "rc=$?" >> gpurun_out/${P}_c4_e2e_gaps.err
timeout 600 python -m pytest tests/test_gpu_prefix.py -x -q > gpurun_out/${P}_pytest_prefix.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_prefix.log
timeout 300 python tools/prefix_phases.py c1 c2 c3 --algo 5 > gpurun_out/${P}_adapt.jsonl 2>&1
