"""BASELINE.json configs[4] (c5: l = 4096, 8 functions, eps 1e-12) end to end
on ONE GPU by streaming the order shards.

The c5 plan set (~0.2-0.3 TB) does not fit one B200, so the config is quoted
on 2/4/8 GPUs with the orders sharded.  With one GPU per call
this script runs exactly the per-rank work of a W-way order sharding, one rank
after the other on the same device: for every order range the plans are built
(GPU plan builder), packed and uploaded as an order-range transform
(SHT.range = what bfly_shard_create holds per rank), the Legendre stage writes
the range's bins of the [bin][b][t] exchange buffer (the m <-> theta transpose
is then a no-op: all "ranks" share the buffer), and the plans are dropped
again.  The phi stage (length 4l - 1 = 16383) runs once over all bins.
Analysis is the reverse with the plans rebuilt.  Nothing here waits on another
rank's kernel; the per-range Legendre times are the per-rank order-side times
of the sharded run and are reported as such.

Checks: analysis(synthesis(beta)) = beta (relative l2 per member and overall),
and -- with --oracle -- the Legendre stage of sampled
orders against the reference's own plans (CPU oracle, oracle/_ref).

    python scripts/c5_streamed.py [--l 4096] [--batch 8] [--shards 8] [--eps 1e-12] [--oracle]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from oracle import sht_oracle  # noqa: E402  (seeded inputs, optional CPU check)
from paper_0910_5435_b200.sharded import coefficient_slices, partition_orders  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--l", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--eps", type=float, default=1e-12)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    l, B, W, eps = args.l, args.batch, args.shards, args.eps
    N = 4 * l - 1
    dev = torch.device("cuda", 0)
    ranges = partition_orders(l, W)
    beta_h = sht_oracle.random_coefficients(l, B, seed=1005)
    beta = torch.from_numpy(beta_h).to(dev)
    bins = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device=dev)
    res = {"l": l, "batch": B, "eps": eps, "shards": W, "ranges": ranges, "per_shard": []}

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()  # warm-up (scratch allocation)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    # ---- synthesis: every shard's Legendre stage, then the phi stage -----------
    last = None
    for r, (a, b) in enumerate(ranges):
        t0 = time.perf_counter()
        part = bb.SHT.range(l, a, b, eps=eps)
        build_s = time.perf_counter() - t0
        info = part.info()
        ms = timed(lambda: part.legendre_synthesize(beta, out=bins))
        res["per_shard"].append({"rank": r, "orders": [a, b], "build_s": round(build_s, 1),
                                 "stored_words": info["stored_words"], "legendre_synth_ms": ms,
                                 "mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1)})
        print(json.dumps(res["per_shard"][-1]), file=sys.stderr, flush=True)
        if last is not None:
            del last
        last = part
        torch.cuda.empty_cache()
    grid = torch.empty((B, 2 * l, N), dtype=torch.complex128, device=dev)
    res["phi_synth_ms"] = timed(lambda: last.phi_synthesize(bins, out=grid))
    # ---- analysis: phi stage, then every shard's transposed Legendre stage ----
    res["phi_anal_ms"] = timed(lambda: last.phi_analyze(grid, out=bins))
    del grid
    back = torch.zeros_like(beta)
    for r, (a, b) in enumerate(ranges):
        if r == W - 1:
            part = last
        else:
            t0 = time.perf_counter()
            part = bb.SHT.range(l, a, b, eps=eps)
            res["per_shard"][r]["rebuild_s"] = round(time.perf_counter() - t0, 1)
        ms = timed(lambda: part.legendre_analyze(bins, out=back))
        res["per_shard"][r]["legendre_anal_ms"] = ms
        print(json.dumps({"rank": r, "legendre_anal_ms": ms}), file=sys.stderr, flush=True)
        if part is not last:
            del part
            torch.cuda.empty_cache()
    nrm = torch.linalg.vector_norm
    res["round_trip_rel_l2"] = float((nrm(back - beta) / nrm(beta)).item())
    res["round_trip_rel_l2_per_member"] = [float((nrm(back[i] - beta[i]) / nrm(beta[i])).item()) for i in range(B)]
    words = sum(s["stored_words"] for s in res["per_shard"])
    res["stored_words"] = words
    res["plan_bytes_gb"] = round(8 * words / 1e9, 1)
    syn = [s["legendre_synth_ms"] for s in res["per_shard"]]
    ana = [s["legendre_anal_ms"] for s in res["per_shard"]]
    res["one_gpu_streamed_step_ms"] = sum(syn) + sum(ana) + res["phi_synth_ms"] + res["phi_anal_ms"]
    res["one_gpu_streamed_pairs_per_s"] = B / (res["one_gpu_streamed_step_ms"] * 1e-3)
    # the W-GPU run these shards belong to: the slowest rank's order side, 1/W of the phi stage, and the
    # exchange at NVLink rate (16 B 2l N (W-1)/W bytes per direction in total, 900 GB/s per GPU and direction)
    xchg_ms = 16.0 * B * 2 * l * N * (W - 1) / W / W / 900e9 * 1e3
    res["projection"] = {
        "legendre_max_ms": [max(syn), max(ana)], "legendre_mean_ms": [sum(syn) / W, sum(ana) / W],
        "phi_per_rank_ms": [res["phi_synth_ms"] / W, res["phi_anal_ms"] / W], "exchange_ms_per_direction": xchg_ms,
        "step_ms_no_overlap": max(syn) + max(ana) + (res["phi_synth_ms"] + res["phi_anal_ms"]) / W + 2 * xchg_ms,
    }
    res["projection"]["pairs_per_s"] = B / (res["projection"]["step_ms_no_overlap"] * 1e-3)
    res["projection"]["efficiency_vs_streamed_one_gpu"] = (
        res["one_gpu_streamed_step_ms"] / W / res["projection"]["step_ms_no_overlap"])

    if args.oracle:
        # sampled orders against the reference (its plans, its apply) on the same coefficients
        from oracle import ref as oref
        errs = {}
        for mu0, mu1 in ((0, 2), (l - 1, l + 1), (2 * l - 2, 2 * l)):
            rs = oref.RefPlanSet(l, eps, mu_range=(mu0, mu1))
            rsht = sht_oracle.RefSHT(l, eps, planset=rs)
            bsel = torch.tensor(rsht.range_bins(), device=dev)
            sl = coefficient_slices(l, mu0, mu1)
            bh = np.zeros((B, 4 * l * l), dtype=np.complex128)
            for a, b in sl:
                bh[:, a:b] = beta_h[:, a:b]
            g_ref = rsht.legendre_synthesis_bins(bh)  # (B, 2l, nbins)
            part = bb.SHT.range(l, mu0, mu1, eps=eps, rule=(rsht.nodes, rsht.rho))
            gout = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device=dev)
            part.legendre_synthesize(beta, out=gout)
            got = gout[bsel].permute(1, 2, 0).cpu().numpy()
            errs[f"synth[{mu0},{mu1})"] = float(np.linalg.norm(got - g_ref) / np.linalg.norm(g_ref))
            del part, gout
        res["oracle_rel_l2"] = errs
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
