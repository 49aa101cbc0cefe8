#!/usr/bin/env python3
"""K1 (sketch build) roofline probe on the C2 collection: mean device ms per launch, L2 flushed."""
import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
from paper_1711_07295_b200 import load_library, datasets as D, ssjoin as S
lib = load_library(); coll = D.c2(lib); S.pin_device(coll, 0)
t, o = coll.csr(); n = len(o) - 1
for bits in (64, 128, 256):
    ms = C.c_double(); lib.ssjb_time_build(coll.handle, 1, bits, 0, 0, 20, C.byref(ms))
    b = 4 * len(t) + 8 * (n + 1) + bits // 8 * n
    print(bits, "%.4f ms %.0f GB/s" % (ms.value, b / ms.value / 1e6))
