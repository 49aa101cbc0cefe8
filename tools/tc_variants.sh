#!/bin/bash
# Filter-kernel variant sweep on C2 (b=128): pipeline-only (SSJB_TC_DEBUG=1) and full.
for V in "i8 256" "i8 128" "fp4 192" "fp4 128"; do
  set -- $V
  for DBG in 1 0; do
    SSJB_TC_DEBUG=$DBG SSJB_TC_KIND=$1 SSJB_TC_N=$2 timeout 300 python tools/c2_phases.py 128 2 > gpurun_out/var.jsonl 2>&1
    python - "$1" "$2" "$DBG" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("gpurun_out/var.jsonl")]
f = {r["tau"]: r["ms"]["filter"] for r in rows}
print(sys.argv[1], sys.argv[2], "debug" if sys.argv[3] == "1" else "full ", " ".join(f"{k}:{v:.3f}" for k, v in f.items()),
      "sum %.2f" % sum(f.values()))
PY
  done
done
