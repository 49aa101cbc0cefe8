#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02x}
timeout 300 python tools/heavy_phases.py C4 C5 C3 2>&1 | cut -c1-420 > gpurun_out/${P}_heavy.jsonl
timeout 300 python bench.py --workload c2 --steps 5 --warmup 2 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 value', d['value'], 'e2e', d['e2e']['value'])" >> gpurun_out/${P}_heavy.jsonl 2>&1
for D in 1 5; do SSJB_TC_DEBUG=$D timeout 300 python tools/heavy_phases.py C4 2>&1 | cut -c1-300 >> gpurun_out/${P}_probe.jsonl; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_join or overflow or random or level3 or streamed or sketch" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
timeout 600 python -m pytest tests/test_gpu_heavy.py -x -q -s -k "not sharded" > gpurun_out/${P}_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_heavy_tests.log
