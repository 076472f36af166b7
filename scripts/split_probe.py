"""Time the full transform pair of one configuration (diagnostics; env selects
the program kind, e.g. BFLY_SPLIT=1 BFLY_ROOTS=mma).

usage: python scripts/split_probe.py L B [steps]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from oracle import sht_oracle  # noqa: E402

l, B = int(sys.argv[1]), int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
t0 = time.time()
sht = bb.SHT(l, eps=1e-12)
build = time.time() - t0
beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=5, decaying_member=B - 1)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
grid = sht.synthesize(beta)
back = sht.analyze(grid)
err = (torch.linalg.vector_norm(back - beta) / torch.linalg.vector_norm(beta)).item()
ts, tsyn = [], []
for k in range(steps):
    flush.fill_(k)
    a, m, b = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    sht.synthesize(beta, out=grid)
    m.record()
    sht.analyze(grid, out=back)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
    tsyn.append(a.elapsed_time(m))
step = min(ts)
print(json.dumps({"l": l, "B": B, "env": {k: v for k, v in os.environ.items() if k.startswith("BFLY_")},
                  "step_ms": round(step, 3), "synth_ms": round(min(tsyn), 3), "pairs_s": round(B / step * 1e3, 2),
                  "rt": err, "build_s": round(build, 1), "info": sht.info(), "program": sht.program_info()}), flush=True)
