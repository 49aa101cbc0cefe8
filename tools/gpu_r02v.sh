#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02v}
timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-secondary > gpurun_out/${P}_bench.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/${P}_bench.json').read().strip().splitlines()[-1])
print('C4 value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'cold', d['e2e_cold'])" > gpurun_out/${P}_summary.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_delivery.py tests/test_capi_client.py -x -q -k "not random" > gpurun_out/${P}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_tests.log
