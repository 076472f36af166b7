"""Graph program (one persistent launch per direction) at several plan-group
sizes: Legendre-stage time per direction and the full step, event-timed;
agreement across group sizes (bit-identical expected).

    python scripts/graph_timing.py L B [group ...]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from oracle import sht_oracle  # noqa: E402


def timed(sht, beta, K=5):
    grid = sht.synthesize(beta)
    back = sht.analyze(grid)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    for k in range(K):
        flush.fill_(k)
        ev[k][0].record()
        sht.synthesize(beta, out=grid)
        ev[k][1].record()
        sht.analyze(grid, out=back)
        ev[k][2].record()
    torch.cuda.synchronize()
    syn = sum(e[0].elapsed_time(e[1]) for e in ev) / K
    ana = sum(e[1].elapsed_time(e[2]) for e in ev) / K
    sht.engine_time(True)
    for k in range(K):
        flush.fill_(k)
        sht.synthesize(beta, out=grid)
        sht.analyze(grid, out=back)
    torch.cuda.synchronize()
    ms, n = sht.engine_time(False)
    return grid, back, {"synth_ms": syn, "anal_ms": ana, "pairs_per_s": beta.shape[0] / ((syn + ana) * 1e-3),
                        "legendre_ms": [ms[0] / K, ms[1] / K]}


def main():
    l, B = int(sys.argv[1]), int(sys.argv[2])
    groups = [int(x) for x in sys.argv[3:]] or [4096]
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=99)).cuda()
    res = {"l": l, "B": B}
    os.environ["BFLY_WAVES"] = "1"
    g0 = b0 = None
    flops = None
    for g in groups:
        os.environ["BFLY_GRAPH_GROUP"] = str(g)
        t0 = time.time()
        gr = bb.SHT(l, eps=1e-12)
        build = time.time() - t0
        if flops is None:
            flops = 2 * 4 * B * gr.info()["stored_words"]
            res["build_s"] = build
            res["program"] = gr.program_info()
        g1, b1, r = timed(gr, beta)
        r["tflops"] = [flops / (t * 1e-3) / 1e12 for t in r["legendre_ms"]]
        if g0 is None:
            g0, b0 = g1.clone(), b1.clone()
        r["synth_vs_first"] = float((torch.linalg.vector_norm(g1 - g0) / torch.linalg.vector_norm(g0)).item())
        r["anal_vs_first"] = float((torch.linalg.vector_norm(b1 - b0) / torch.linalg.vector_norm(b0)).item())
        r["round_trip"] = float((torch.linalg.vector_norm(b1 - beta) / torch.linalg.vector_norm(beta)).item())
        res[f"graph_{g}"] = r
        del gr
        torch.cuda.empty_cache()
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
