#!/bin/bash
# Filter flavour sweep on C2 (b=128 and 256): per-tau filter ms for
# int8 / fp4 tensor-core kernels with the level-2 GEMM forced on/off/auto.
mkdir -p gpurun_out
for BITS in 128 256; do
for V in "i8 auto" "i8 0" "i8 1" "fp4 0"; do
  set -- $V
  if [ "$2" = auto ]; then unset SSJB_L2GEMM; else export SSJB_L2GEMM=$2; fi
  SSJB_TC_KIND=$1 timeout 300 python tools/c2_phases.py $BITS 3 > gpurun_out/var.jsonl 2>&1
  python - "$1" "$2" "$BITS" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("gpurun_out/var.jsonl") if l.startswith("{")]
f = {r["tau"]: (r["ms"]["filter"], r["ms"]["verify"], r["kernel"]) for r in rows}
print("b=%s %s l2=%s" % (sys.argv[3], sys.argv[1], sys.argv[2]), " ".join(f"{k}:{v[0]:.3f}/{v[1]:.3f}/k{v[2]}" for k, v in f.items()),
      "sum %.2f" % sum(v[0] + v[1] for v in f.values()), flush=True)
PY
done
done
