"""Order-sharding projection at c3 (l=1024, 16 functions) from one GPU (diagnostics).

Each rank's order-side work of the sharded transform: the
Legendre stage of its order range, including the parity combine / split into
the exchange layout, is run for real -- rank after rank on this GPU through
SHT.range handles (the stage-wise entry points) -- and timed with CUDA events.
The slab-side phi stage splits the grid rows evenly, so its time is the
single-GPU phi time / W (given on the command line, from the ncu summary); the
all-to-all moves 16 B x B x 2l x (4l-1) x (W-1)/W^2 per GPU and direction at an
assumed per-GPU NVLink rate.  Nothing here waits on another rank.

usage: python scripts/shard_projection.py [W,...] [phi_ms_per_step] [nvlink_GBps]"""
import gc
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from paper_0910_5435_b200.sharded import partition_orders  # noqa: E402

l, B = 1024, 16
Ws = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8").split(",")]
phi_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 6.33
link = float(sys.argv[3]) if len(sys.argv) > 3 else 700.0
N = 4 * l - 1
g = torch.Generator(device="cuda").manual_seed(11)
beta = torch.complex(torch.randn((B, 4 * l * l), dtype=torch.float64, device="cuda", generator=g),
                     torch.randn((B, 4 * l * l), dtype=torch.float64, device="cuda", generator=g))
gd = torch.complex(torch.randn((N, B, 2 * l), dtype=torch.float64, device="cuda", generator=g),
                   torch.randn((N, B, 2 * l), dtype=torch.float64, device="cuda", generator=g))


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


out = {"l": l, "B": B, "phi_ms_single_gpu": phi_ms, "nvlink_GBps_assumed": link, "W": {}}
for W in Ws:
    per = []
    for r, (a, b) in enumerate(partition_orders(l, W)):
        sht = bb.SHT.range(l, a, b, eps=1e-12, threads=os.cpu_count())
        bins = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device="cuda")
        cf = torch.zeros_like(beta)
        ts = timed(lambda: sht.legendre_synthesize(beta, out=bins))
        ta = timed(lambda: sht.legendre_analyze(gd, out=cf))
        per.append({"orders": [a, b], "legendre_synth_ms": ts, "legendre_anal_ms": ta})
        del sht, bins, cf
        gc.collect()
        torch.cuda.empty_cache()
    order_side = max(p["legendre_synth_ms"] + p["legendre_anal_ms"] for p in per)
    a2a_ms = 2 * 16.0 * B * 2 * l * N * (W - 1) / W ** 2 / (link * 1e9) * 1e3
    step = order_side + phi_ms / W + a2a_ms
    out["W"][W] = {"ranks": per, "order_side_ms_max": order_side, "phi_ms": phi_ms / W, "all_to_all_ms": a2a_ms,
                   "projected_step_ms": step}
    print(json.dumps({"W": W, "order_side_ms_max": round(order_side, 3), "phi_ms": round(phi_ms / W, 3),
                      "all_to_all_ms": round(a2a_ms, 3), "projected_step_ms": round(step, 3)}), flush=True)
print(json.dumps(out))
