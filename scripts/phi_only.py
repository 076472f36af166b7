"""The fused phi stage alone (bfly_phi_time): python scripts/phi_only.py L B [iters]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0910_5435_b200._lib import check, lib  # noqa: E402

l, B = int(sys.argv[1]), int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
ms = (C.c_double * 2)()
check(lib().bfly_phi_time(l, B, iters, ms))
N = 4 * l - 1
hbm = 2 * 16 * B * 2 * l * N  # grid once + chain values once (about the same size)
print(json.dumps({"l": l, "B": B, "ms": [ms[0], ms[1]], "hbm_bound_ms": hbm / 6.5e12 * 1e3}))
