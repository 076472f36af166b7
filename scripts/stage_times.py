"""Per-stage device times of one configuration through the stage-wise entry
points (diagnostics): Legendre synthesis (coefficients -> phi bins), phi
synthesis (cuFFT), phi analysis, Legendre analysis; plus the fused full
transforms when available.  CUDA events, L2 flushed before each stage.

usage: python scripts/stage_times.py L B [reps]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402

l, B = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
t0 = time.time()
sht = bb.SHT(l, eps=1e-12, threads=os.cpu_count())
build = time.time() - t0
g = torch.Generator(device="cuda").manual_seed(7)
beta = torch.complex(torch.randn((B, 4 * l * l), dtype=torch.float64, device="cuda", generator=g),
                     torch.randn((B, 4 * l * l), dtype=torch.float64, device="cuda", generator=g))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    ts = []
    for k in range(reps):
        flush.fill_(k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return r, min(ts)


bins, t_ls = timed(lambda: sht.legendre_synthesize(beta))
grid, t_ps = timed(lambda: sht.phi_synthesize(bins))
gd, t_pa = timed(lambda: sht.phi_analyze(grid))
back, t_la = timed(lambda: sht.legendre_analyze(gd))
err = (torch.linalg.vector_norm(back - beta) / torch.linalg.vector_norm(beta)).item()
out = {"l": l, "B": B, "build_s": round(build, 1), "legendre_synth_ms": t_ls, "phi_synth_ms": t_ps,
       "phi_anal_ms": t_pa, "legendre_anal_ms": t_la, "rt_stagewise": err}
try:
    _, t_fs = timed(lambda: sht.synthesize(beta, out=grid))
    _, t_fa = timed(lambda: sht.analyze(grid, out=back))
    out.update(full_synth_ms=t_fs, full_anal_ms=t_fa, pairs_s=B / (t_fs + t_fa) * 1e3)
except Exception as e:  # noqa: BLE001
    out["full"] = str(e)
print(json.dumps(out), flush=True)
