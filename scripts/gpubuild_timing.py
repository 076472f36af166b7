"""Time the GPU plan builder on a full GL-row plan set:
python scripts/gpubuild_timing.py L EPS [MU0 MU1]  (JSON line on stdout)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402

l = int(sys.argv[1])
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-12
mu0, mu1 = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 2 * l)
os.environ.setdefault("BFLY_BUILD_VERBOSE", "1")
t0 = time.perf_counter()
plans = bb.build_glrow_planset(l, eps, mu_range=(mu0, mu1))
dt = time.perf_counter() - t0
info = [p.info() for p in plans]
print(json.dumps({"l": l, "eps": eps, "mu": [mu0, mu1], "plans": len(plans), "build_s": dt,
                  "stored_words": sum(i["stored_words"] for i in info),
                  "levels_max": max(i["levels"] for i in info), "k_max": max(i["k_max"] for i in info),
                  "builder": os.environ.get("BFLY_BUILDER", "auto")}))
