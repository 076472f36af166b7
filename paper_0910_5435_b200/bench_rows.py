"""GPU mode of the reference CLI's ``bfly bench``.

The reference times one 1-D butterfly transform per row and prints the
paper-table CSV schema (``tools/bfly_main.cpp:99-150`` builds and times a row,
``:166-183`` prints it)::

    n,m,parity,k_max,k_avg,k_sigma,t_dir,t_fwd,t_inv,t_quad,t_comp,m_max,eps_fwd,eps_inv

This module reads plans the reference built and saved (``bfly plan build`` ->
BFLY1 files, ``include/bfly/serialize.hpp:14-31``), applies them on the GPU
one vector per call like the reference's ``time_call`` (``tools/bfly_main.cpp:
48-60``: a warm-up call, then repetitions until at least 0.05 s; device time by
CUDA events around the repetitions, device-resident vectors) and prints the
same columns.  Columns that need the reference's quadrature or dense matrix
or its build timings (t_dir, t_quad, t_comp, eps_fwd) are "NA", as the reference
prints when it skips them; eps_inv is the worst max-abs round
trip error of apply_transpose(apply(v)) over unit test vectors (the reference's
definition, :143-148).  BFLY1 carries no order / parity, so they come from the
command line (default NA).

    python -m paper_0910_5435_b200.bench_rows plan.bfly1 [...] [--m 3 --parity odd]
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

from .butterfly import ButterflyPlan

HEADER = "n,m,parity,k_max,k_avg,k_sigma,t_dir,t_fwd,t_inv,t_quad,t_comp,m_max,eps_fwd,eps_inv"
TEST_VECTORS = 4  # the reference's kTestVectors


def _fmt(x: float | None) -> str:
    return "NA" if x is None else f"{x:.3e}"


def _time_call(fn, min_seconds: float = 0.05) -> float:
    """Seconds per call on the device (CUDA events), after one warm-up call."""
    import torch
    fn()
    torch.cuda.synchronize()
    reps, total = 1, 0.0
    while True:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        total = a.elapsed_time(b) * 1e-3
        if total >= min_seconds or reps >= 1 << 20:
            return total / reps
        reps *= 2


def bench_row(plan: ButterflyPlan, m: str = "NA", parity: str = "NA", seed: int = 1) -> str:
    """One CSV row for a square butterfly plan (the reference bench's plans are n x n)."""
    import torch
    info = plan.info()
    n_rows, n_cols = info["n_rows"], info["n_cols"]
    ps = plan.device_set(0)
    rng = np.random.default_rng(seed)
    vs = []
    for _ in range(TEST_VECTORS):
        v = rng.uniform(-1.0, 1.0, n_cols)
        vs.append(torch.from_numpy(v / np.linalg.norm(v)).cuda())
    y = torch.empty(n_rows, dtype=torch.float64, device="cuda")
    x = torch.empty(n_cols, dtype=torch.float64, device="cuda")
    t_fwd = _time_call(lambda: ps.apply_device(vs[0], y, 1, False))
    w = torch.from_numpy(rng.uniform(-1.0, 1.0, n_rows)).cuda()
    t_inv = _time_call(lambda: ps.apply_device(w, x, 1, True))
    eps_inv = 0.0
    for v in vs:
        ps.apply_device(v, y, 1, False)
        ps.apply_device(y, x, 1, True)
        eps_inv = max(eps_inv, float((x - v).abs().max().item()))
    return ",".join([str(n_cols), str(m), str(parity), str(info["k_max"]), f"{info['k_avg']:.1f}",
                     f"{info['k_sigma']:.1f}", "NA", _fmt(t_fwd), _fmt(t_inv), "NA", "NA",
                     str(info["m_max_words"]), "NA", _fmt(eps_inv)])


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("plans", nargs="+", help="BFLY1 plan files (reference `bfly plan build`)")
    ap.add_argument("--m", nargs="*", default=None, help="order per plan (default NA)")
    ap.add_argument("--parity", nargs="*", default=None, help="even / odd per plan (default NA)")
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args(argv)
    ms = args.m or ["NA"] * len(args.plans)
    pars = args.parity or ["NA"] * len(args.plans)
    if len(ms) != len(args.plans) or len(pars) != len(args.plans):
        ap.error("--m / --parity need one value per plan")
    print(HEADER)
    for path, m, par in zip(args.plans, ms, pars):
        with open(path, "rb") as f:
            plan = ButterflyPlan.from_bfly1(f.read())
        print(bench_row(plan, m, par, args.seed), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
