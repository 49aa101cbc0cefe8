#!/usr/bin/env python3
"""K1 (sketch build) roofline probe: mean device ms per launch with L2 flushed
(ssjb_time_build), on the C2 collection and, with an argument, on C4/C5.

    python tools/k1_probe.py [C4|C5]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import load_library, ssjoin as S  # noqa: E402

lib = load_library()
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
coll = {"C2": D.c2, "C4": D.c4, "C5": D.c5}[name](lib)
S.pin_device(coll, 0)
t, o = coll.csr()
n = len(o) - 1
for bits in (64, 128, 256):
    ms = C.c_double()
    lib.ssjb_time_build(coll.handle, 1, bits, 0, 0, 20, C.byref(ms))
    b = 4 * len(t) + 8 * (n + 1) + bits // 8 * n
    print(f"{name} b={bits}: {ms.value:.4f} ms, {b / 1e6:.1f} MB, {b / ms.value / 1e6:.0f} GB/s", flush=True)
