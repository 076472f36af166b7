"""Minimal repro: every GL-row plan of one bandlimit in one engine launch, both directions."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0910_5435_b200 as bb

l = int(sys.argv[1]) if len(sys.argv) > 1 else 256
direction = sys.argv[2] if len(sys.argv) > 2 else "both"
plans = bb.build_glrow_planset(l, 1e-12)
ps = bb.PlanSet(plans)
print("info", ps.info(), flush=True)
rng = np.random.default_rng(0)
nrhs = 4
if direction in ("fwd", "both"):
    x = rng.standard_normal(sum(ps.cols) * nrhs)
    y = ps.apply_host(x, nrhs, False)
    print("fwd ok", np.linalg.norm(y), flush=True)
if direction in ("bwd", "both"):
    w = rng.standard_normal(sum(ps.rows) * nrhs)
    z = ps.apply_host(w, nrhs, True)
    print("bwd ok", np.linalg.norm(z), flush=True)
