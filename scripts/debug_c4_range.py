"""Diagnose GPU vs reference differences on one order range at large l:
per plan (plan-set apply, R right-hand sides) and per bin / member chunk /
row block of the SHT Legendre stage (SHT.range on the reference's plans)."""
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from oracle import ref, sht_oracle  # noqa: E402
from paper_0910_5435_b200.sharded import coefficient_slices  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    l = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    mu0, mu1 = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 8)
    eps = 1e-12
    t0 = time.time()
    rs = ref.RefPlanSet(l, eps, mu_range=(mu0, mu1))
    print(f"ref build {time.time() - t0:.1f}s, {len(rs)} plans", flush=True)
    plans = [bb.ButterflyPlan.from_bfly1(rs.plan(i).save()) for i in range(len(rs))]
    for i, (mu, p) in enumerate(rs.keys):
        info = rs.plan(i).info()
        print("plan", mu, p, info, flush=True)
    ps = bb.PlanSet(plans)
    rng = np.random.default_rng(1)
    for nrhs in (1, 4, 16, 64, 128, 256):
        ins = [rng.standard_normal((p.n_cols, nrhs)) for p in plans]
        flat, _ = ps.stack(ins)
        got = ps.unstack(ps.apply_host(flat, nrhs, False), nrhs, False)
        want, _ = rs.apply_all(ins, transpose=False)
        errs = [rel(g, w) for g, w in zip(got, want)]
        worst = int(np.argmax(errs))
        colerr = [rel(got[worst][:, c], want[worst][:, c]) for c in range(nrhs)]
        rowblk = [rel(got[worst][r:r + 128], want[worst][r:r + 128]) for r in range(0, l, 128)]
        print(f"planset fwd nrhs={nrhs}: max {max(errs):.3e} at plan {rs.keys[worst]}; worst cols "
              f"{np.argsort(colerr)[-4:].tolist()} {sorted(colerr)[-4:]}; row blocks {['%.1e' % e for e in rowblk]}",
              flush=True)
        wins = [rng.standard_normal((l, nrhs)) for _ in plans]
        flat, _ = ps.stack(wins)
        got = ps.unstack(ps.apply_host(flat, nrhs, True), nrhs, True)
        want, _ = rs.apply_all(wins, transpose=True)
        errs = [rel(g, w) for g, w in zip(got, want)]
        print(f"planset bwd nrhs={nrhs}: max {max(errs):.3e}", flush=True)
    # SHT Legendre stage on the range
    sht_ref = sht_oracle.RefSHT(l, eps, planset=rs)
    bins = sht_ref.range_bins()
    N = 4 * l - 1
    for B in (1, 16, 64):
        beta = np.zeros((B, 4 * l * l), dtype=np.complex128)
        slices = coefficient_slices(l, mu0, mu1)
        for a, b in slices:
            beta[:, a:b] = rng.standard_normal((B, b - a)) + 1j * rng.standard_normal((B, b - a))
        g_ref = sht_ref.legendre_synthesis_bins(beta)
        sht = bb.SHT.range(l, mu0, mu1, eps=eps, plans=plans)
        dev = torch.device("cuda", 0)
        beta_d = torch.zeros((B, 4 * l * l), dtype=torch.complex128, device=dev)
        for a, b in slices:
            beta_d[:, a:b] = torch.from_numpy(np.ascontiguousarray(beta[:, a:b])).to(dev)
        gout = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device=dev)
        sht.legendre_synthesize(beta_d, out=gout)
        got = gout[torch.tensor(bins, device=dev)].permute(1, 2, 0).cpu().numpy()
        per_bin = [rel(got[:, :, j], g_ref[:, :, j]) for j in range(len(bins))]
        per_mem = [rel(got[b], g_ref[b]) for b in range(B)]
        print(f"SHT synth B={B} waves={sht.uses_waves(B)}: total {rel(got, g_ref):.3e}; per bin "
              f"{dict(zip(bins, ['%.1e' % e for e in per_bin]))}; worst members {np.argsort(per_mem)[-4:].tolist()} "
              f"{['%.1e' % e for e in sorted(per_mem)[-4:]]}", flush=True)
        j = int(np.argmax(per_bin))
        rb = [rel(got[:, r:r + 128, j], g_ref[:, r:r + 128, j]) for r in range(0, 2 * l, 128)]
        print("   worst bin row blocks", ['%.1e' % e for e in rb], flush=True)
        del gout, beta_d, sht
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
