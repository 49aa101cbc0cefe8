#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02y}
for V in default tcmold default tcmold; do
  if [ $V = default ]; then unset SSJB_LIB; else export SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_$V.so; fi
  echo "== $V" >> gpurun_out/${P}_c2.txt
  timeout 300 python tools/c2_phases.py 128 3 2>&1 | python -c "
import json,sys
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print(' '.join(f\"{r['tau']}:{r['ms']['filter']:.3f}/k{r['kernel']}\" for r in rows), 'sum_filter %.2f' % sum(r['ms']['filter'] for r in rows))" >> gpurun_out/${P}_c2.txt
  timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 value', d['value'], 'e2e', d['e2e']['value'])" >> gpurun_out/${P}_c2.txt 2>&1
done
