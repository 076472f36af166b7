"""BASELINE.json configs[3] on one GPU: l=2048, batch 64, eps 1e-12 (or --eps).

Seeded N(0,1) complex coefficients generated on the device (17 GB per batch;
the oracle cannot run this size, so the checks are the size-independent
properties: analysis(synthesis(beta)) = beta and linearity on two members).
Prints one JSON line: plan build time, device-resident pairs/s over --steps,
round-trip relative l2, memory high-water mark."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--l", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--eps", type=float, default=1e-12)
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    l, B = args.l, args.batch
    t0 = time.perf_counter()
    sht = bb.SHT(l, eps=args.eps, threads=os.cpu_count())
    build_s = time.perf_counter() - t0
    info = sht.info()
    g = torch.Generator(device="cuda").manual_seed(2048)
    beta = torch.complex(torch.randn((B, 4 * l * l), dtype=torch.float64, device="cuda", generator=g),
                         torch.randn((B, 4 * l * l), dtype=torch.float64, device="cuda", generator=g))
    # coefficients outside the bandlimit's triangle (k < |m|) do not exist in the
    # packed layout, so every entry is a real coefficient
    grid = torch.empty((B, 2 * l, 4 * l - 1), dtype=torch.complex128, device="cuda")
    back = torch.empty_like(beta)
    sht.synthesize(beta, out=grid)  # warm-up (cuFFT plans, scratch)
    sht.analyze(grid, out=back)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        sht.synthesize(beta, out=grid)
        sht.analyze(grid, out=back)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    rt = (torch.linalg.vector_norm(back - beta) / torch.linalg.vector_norm(beta)).item()
    g2 = sht.synthesize(2.5 * beta[:1] + beta[1:2])
    lin = (torch.linalg.vector_norm(g2 - (2.5 * grid[:1] + grid[1:2])) / torch.linalg.vector_norm(g2)).item()
    step = sum(ts) / len(ts)
    print(json.dumps({"l": l, "batch": B, "eps": args.eps, "plan_build_s": round(build_s, 1),
                      "stored_words": info["stored_words"], "step_ms": round(step, 1),
                      "pairs_s": round(B / step * 1e3, 2), "round_trip_rel_l2": rt, "linearity_rel_l2": lin,
                      "max_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
                      "scratch_gb_env": os.environ.get("BFLY_SCRATCH_GB")}))


if __name__ == "__main__":
    main()
