"""CPU checks of the wave-program compiler (no GPU needed).

tests/wave_emulator.py replays the level-synchronous program build_waves
compiles (the batched path's node list, levels, transposed pairs, root stripes;
fetched through bfly_waves_inspect) with the tensor-core kernels' semantics in
numpy on a NaN-poisoned V; its results must equal the reference's
bfly::apply / apply_transpose (src/butterfly.cpp:384-513) on the same plans.
This pins the compiler independently of the CUDA kernels, which the GPU tests
check against the whole-chain engine and the reference.
"""
import numpy as np
import pytest

import paper_0910_5435_b200 as bb
from wave_emulator import WaveProgram


def kernel_matrix(n):
    i = np.arange(n)[:, None] + 0.5
    j = np.arange(n)[None, :] + 0.5
    return np.cos(8.0 * np.pi * i * j / n) / np.sqrt(n)


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def check(ref_plans, R=5, tol=1e-14):
    plans = [bb.ButterflyPlan.from_bfly1(p.save()) for p in ref_plans]
    prog = WaveProgram(plans)
    rng = np.random.default_rng(17)
    ins = [rng.standard_normal((p.n_cols, R)) for p in plans]
    for g, rp, x in zip(prog.apply(ins), ref_plans, ins):
        assert np.all(np.isfinite(g)), "read of an unwritten cell"
        assert relerr(g, rp.apply(x)) <= tol
    wins = [rng.standard_normal((p.n_rows, R)) for p in plans]
    for g, rp, w in zip(prog.apply_transpose(wins), ref_plans, wins):
        assert np.all(np.isfinite(g)), "read of an unwritten cell"
        assert relerr(g, rp.apply_transpose(w)) <= tol
    return prog


@pytest.mark.parametrize("a,eps,c", [
    (np.eye(256), 1e-14, 60),
    (kernel_matrix(300), 1e-13, 60),
    (kernel_matrix(130), 1e-13, 60),
    (kernel_matrix(64), 1e-13, 16),
    (np.random.default_rng(71).uniform(-1, 1, (40, 7)), 1e-13, 60),
])
def test_dense_plans(oracle, a, eps, c):
    check([oracle.RefPlan.dense(a, eps, c)])


@pytest.mark.parametrize("l", [8, 32, 96])
def test_glrow_planset(oracle, l):
    """All (mu, parity) plans of a bandlimit in one wave program; full-rank leaves
    alias their coefficient cells (no node), levels are consistent."""
    rs = oracle.RefPlanSet(l, 1e-12)
    prog = check([rs.plan(i) for i in range(len(rs))])
    levels = [prog.nodes[i]["level"] for i in prog.fwd]
    assert levels == sorted(levels) and (not levels or levels[0] >= 1)
    assert prog.aliased > 0
