#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02j}
for V in default nosusp susp1k lateacc; do
  if [ $V = default ]; then unset SSJB_LIB; else export SSJB_LIB=$PWD/paper_1711_07295_b200/lib/variants/libssjoin_$V.so; fi
  echo "== $V" >> gpurun_out/${P}_variants.txt
  timeout 300 python tools/heavy_phases.py C4 2>&1 | cut -c1-420 >> gpurun_out/${P}_variants.txt
  timeout 300 python bench.py --workload c2 --steps 5 --warmup 2 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 value', d['value'], 'e2e', d['e2e']['value'])" >> gpurun_out/${P}_variants.txt 2>&1
done
unset SSJB_LIB
timeout 900 python -m pytest tests/test_naive_rs.py -x -q -s > gpurun_out/${P}_rs_tests.log 2>&1; echo rc=$? >> gpurun_out/${P}_rs_tests.log
