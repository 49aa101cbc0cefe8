#!/bin/bash
# Level-2 GEMM choice on the C2 sweep: the cutoff factor (SSJB_L2GEMM_FACTOR).
mkdir -p gpurun_out
P=${TAG:-r02s}
for F in 1.25 1.6 2.0 3.0; do
  echo "== factor $F" >> gpurun_out/${P}_c2.txt
  SSJB_L2GEMM_FACTOR=$F timeout 300 python tools/c2_phases.py 128 3 2>&1 | python -c "
import json,sys
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print(' '.join(f\"{r['tau']}:{r['ms']['filter']:.3f}/{r['ms']['verify']:.3f}/k{r['kernel']}/w{r['wall_ms']:.2f}\" for r in rows), 'sum_wall %.2f' % sum(r['wall_ms'] for r in rows))" >> gpurun_out/${P}_c2.txt
  SSJB_L2GEMM_FACTOR=$F timeout 300 python bench.py --workload c2 --steps 5 --warmup 2 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 value', d['value'], 'e2e', d['e2e']['value'])" >> gpurun_out/${P}_c2.txt 2>&1
done
