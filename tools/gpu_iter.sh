#!/bin/bash
# Iteration run: GPU parity, C2 per-tau phases (1-CTA / pair), pair-kernel trace,
# heavy phases, full-size + heavy parity (HEAVY_TESTS=1), e2e bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases128.jsonl 2>&1
SSJB_TC2=1 timeout 300 python tools/c2_phases.py 128 3 > gpurun_out/phases_tc2.jsonl 2>&1
rm -f gpurun_out/tc_trace.txt
SSJB_TC2=1 SSJB_TC_DEBUG=2 timeout 300 python - <<'PY' > gpurun_out/trace_runs.txt 2>&1
import sys
sys.path.insert(0, ".")
import paper_1711_07295_b200 as pkg
from paper_1711_07295_b200 import datasets as D, ssjoin as S
lib = pkg.load_library()
coll = D.c2(lib)
S.pin_device(coll, 0)
for rep in range(2):
    r = S.join(coll, D.c2_options(lib, (7, 10)))
print("filter_ms", r.extra["ms_filter"])
PY
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -n "$HEAVY_TESTS" ]; then
timeout 900 python tools/heavy_phases.py C3 C5 C4 > gpurun_out/heavy_phases.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_heavy.py -x -q -s > gpurun_out/pytest_heavy.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_heavy.log
fi
