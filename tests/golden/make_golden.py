"""Generate the golden fixtures in tests/golden/ from the compiled reference.

Run in the build container (needs /root/reference, which oracle/Makefile
compiles unmodified into oracle/_ref/libbfly_ref.so):

    python tests/golden/make_golden.py

The fixtures let the GPU tests (where /root/reference does not exist) and the
CPU oracle tests check against outputs of the reference itself:

* ``plan_glrow_l32_mu3_p1.bfly1`` — the reference builder's GL-row plan for
  (l=32, mu=3, odd chain) serialised by reference src/serialize.cpp, with
  ``plan_glrow_l32_mu3_p1.npz``: seeded x (n_cols x 4) / w (l x 4), and the
  reference's bfly::apply(x) and apply_transpose(w) (src/butterfly.cpp:384-513).
* ``transform_m3_n64.npz`` — column 17 of the reference transform plan
  (m=3, n=64, even, eps 1e-12) as applied by the reference, plus the dense
  column (the known answer of reference tests/test_cli.cpp:93-123).
* ``rule_l32.npz`` — build_rule(0, 32, even): the 32 positive GL nodes of
  degree 64 and rho = 2 w_GL (src/quadrature.cpp).
* ``sht_l16.npz`` / ``sht_l32.npz`` — seeded coefficients (B=2, member 1
  scaled by (k+1)^-2), the reference-backed synthesis grid and the analysis of
  that grid (reference apply per plan + numpy DFT; oracle/sht_oracle.py).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from oracle.sht_oracle import RefSHT, random_coefficients  # noqa: E402


def main() -> None:
    rng = np.random.default_rng(20260901)

    # one plan, both directions
    p = ref.RefPlan.glrow(32, 3, 1, 1e-12)
    blob = p.save()
    with open(os.path.join(HERE, "plan_glrow_l32_mu3_p1.bfly1"), "wb") as f:
        f.write(blob)
    nr, nc = p.shape
    x = rng.standard_normal((nc, 4))
    w = rng.standard_normal((nr, 4))
    np.savez_compressed(os.path.join(HERE, "plan_glrow_l32_mu3_p1.npz"), x=x, w=w, ax=p.apply(x),
                        atw=p.apply_transpose(w), dense=ref.dense_glrow(32, 3, 1))

    # transform plan, column 17
    t = ref.RefPlan.transform(3, 64, 0, 1e-12)
    e = np.zeros(64)
    e[17] = 1.0
    a, nodes, wts = ref.dense_transform(3, 64, 0)
    np.savez_compressed(os.path.join(HERE, "transform_m3_n64.npz"), col17=t.apply(e), dense_col17=a[:, 17])

    nodes, rho, _ = ref.rule(0, 32, 0)
    np.savez_compressed(os.path.join(HERE, "rule_l32.npz"), nodes=nodes, rho=rho)

    for l, seed in ((16, 1016), (32, 1032)):
        beta = random_coefficients(l, 2, seed, decaying_member=1)
        sht = RefSHT(l, 1e-12)
        grid = sht.synthesize(beta)
        back = sht.analyze(grid)
        np.savez_compressed(os.path.join(HERE, f"sht_l{l}.npz"), beta=beta, grid=grid, back=back,
                            seed=seed, eps=1e-12)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
