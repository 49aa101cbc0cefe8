#!/usr/bin/env python3
"""Run the golden joins one by one under the current SSJB_* environment and
report the first failing fixture (debugging aid for new filter kernels)."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from conftest import golden_collection  # noqa: E402
import paper_1711_07295_b200 as pkg  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

lib = pkg.load_library()
golden = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
arrays = np.load(os.path.join(ROOT, "tests", "golden", "golden_pairs.npz"))
only = sys.argv[1] if len(sys.argv) > 1 else None
for k, e in enumerate(golden["joins"]):
    if only is not None and str(k) != only:
        continue
    coll = S.Collection.from_csr(lib, *golden_collection(arrays, e["collection"]))
    o = S.default_options(lib)
    for key, v in e["options"].items():
        setattr(o, key, v)
    try:
        rep = S.join(coll, o)
    except Exception as ex:  # noqa: BLE001
        print("FAIL", k, e["label"], e["collection"], len(coll), e["options"], ex, flush=True)
        sys.exit(1)
    ok = (len(rep.pairs) == e["pair_count"] and
          hashlib.sha256(rep.pairs.tobytes()).hexdigest() == e["pairs_sha256"] and
          all(rep.counters[c] == e["counters"][c] for c in e["counters"]))
    if not ok:
        print("MISMATCH", k, e["label"], e["collection"], len(coll), e["options"], rep.counters, e["counters"],
              len(rep.pairs), e["pair_count"], flush=True)
        sys.exit(2)
print("all", len(golden["joins"]), "ok")
