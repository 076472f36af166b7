"""Plan-set apply (bfly_dev_apply, the reference's bfly::apply for many
right-hand sides) on the engine vs the wave programs (diagnostics).

usage: python scripts/planset_timing.py L nrhs[,nrhs...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from paper_0910_5435_b200.butterfly import build_glrow_planset  # noqa: E402

l = int(sys.argv[1])
plans = build_glrow_planset(l, 1e-12, 60)
os.environ["BFLY_WAVE_MIN_RHS"] = "1000000"
engine = bb.PlanSet(plans)
os.environ["BFLY_WAVE_MIN_RHS"] = "1"
waves = bb.PlanSet(plans)
cols, rows = sum(p.n_cols for p in plans), sum(p.n_rows for p in plans)
words = sum(p.info()["stored_words"] for p in plans) if hasattr(plans[0], "info") else None
for nrhs in [int(x) for x in sys.argv[2].split(",")]:
    res = {"l": l, "nrhs": nrhs}
    for name, ps in (("engine", engine), ("waves", waves)):
        for tr in (False, True):
            n_in, n_out = (rows, cols) if tr else (cols, rows)
            x = torch.randn(n_in * nrhs, dtype=torch.float64, device="cuda")
            y = torch.empty(n_out * nrhs, dtype=torch.float64, device="cuda")
            ps.apply_device(x, y, nrhs, tr)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ps.apply_device(x, y, nrhs, tr)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[f"{name}_{'T' if tr else 'A'}_ms"] = round(min(ts), 4)
            if name == "engine":
                ref = y.clone()
            else:
                pass
    print(json.dumps(res), flush=True)
