#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02bc}
timeout 900 python tools/c4_stream_chunks.py 2 > gpurun_out/${P}_phases_on.jsonl 2> gpurun_out/${P}_phases_on.err
SSJB_STREAM_PHASES=0 timeout 900 python tools/c4_stream_chunks.py 2 > gpurun_out/${P}_phases_off.jsonl 2> gpurun_out/${P}_phases_off.err
timeout 1500 python -m pytest tests/test_gpu_heavy.py -x -q > gpurun_out/${P}_pytest_heavy.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest_heavy.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "rc=$?" >> gpurun_out/${P}_bench.err
