"""CPU checks of the device-program packer (no GPU needed).

tests/engine_emulator.py replays the packed stage stream with the kernel's
record semantics (bounds-checked, NaN-poisoned arena); its results must equal
the reference's bfly::apply / apply_transpose on the same plans.  This pins
arena lifetimes, assign/accumulate flags and the record order of both
directions independently of the CUDA engine.
"""
import numpy as np
import pytest

import paper_0910_5435_b200 as bb
from engine_emulator import Program, emulate


def kernel_matrix(n):
    i = np.arange(n)[:, None] + 0.5
    j = np.arange(n)[None, :] + 0.5
    return np.cos(8.0 * np.pi * i * j / n) / np.sqrt(n)


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def check_against_reference(oracle, ref_plans, tol=1e-14):
    plans = [bb.ButterflyPlan.from_bfly1(p.save()) for p in ref_plans]
    rng = np.random.default_rng(7)
    ins = [rng.standard_normal((p.n_cols, 4)) for p in plans]
    got, prog = emulate(plans, ins, bwd=False)
    for g, rp, x in zip(got, ref_plans, ins):
        assert np.all(np.isfinite(g)), "read of an unwritten cell"
        assert relerr(g, rp.apply(x)) <= tol
    wins = [rng.standard_normal((p.n_rows, 4)) for p in plans]
    got, _ = emulate(plans, wins, bwd=True)
    for g, rp, w in zip(got, ref_plans, wins):
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
    check_against_reference(oracle, [oracle.RefPlan.dense(a, eps, c)])


@pytest.mark.parametrize("l", [32, 96])
def test_glrow_planset(oracle, l):
    rs = oracle.RefPlanSet(l, 1e-12)
    prog = check_against_reference(oracle, [rs.plan(i) for i in range(len(rs))])
    assert all(b <= 49152 and b % 16 == 0 for b in prog.stage_bytes)


def test_reference_transform_plan(oracle):
    check_against_reference(oracle, [oracle.RefPlan.transform(64, 512, 1, 1e-14)])


def test_stage_bounds_and_smem_budget(oracle):
    rs = oracle.RefPlanSet(128, 1e-12)
    plans = [bb.ButterflyPlan.from_bfly1(rs.plan(i).save()) for i in range(len(rs))]
    prog = Program(plans)
    assert max(prog.stage_bytes) <= 49152
    assert prog.smem_bytes <= 227 * 1024
    for s in range(len(prog.stage_bytes)):
        prog.stage(s)  # header consistency


@pytest.mark.parametrize("l", [32, 96])
def test_split_programs(oracle, l):
    """SHT compilation: event program + root program exchanging vectors through C."""
    from engine_emulator import emulate_split
    rs = oracle.RefPlanSet(l, 1e-12)
    plans = [bb.ButterflyPlan.from_bfly1(rs.plan(i).save()) for i in range(len(rs))]
    parity = [p for (_, p) in rs.keys]
    rng = np.random.default_rng(l)
    ins = [rng.standard_normal((p.n_cols, 4)) for p in plans]
    got, (ev, ro) = emulate_split(plans, parity, ins, bwd=False)
    want, _ = rs.apply_all(ins, transpose=False)
    for g, w in zip(got, want):
        assert np.all(np.isfinite(g)) and relerr(g, w) <= 1e-14
    wins = [rng.standard_normal((l, 4)) for _ in plans]
    got, _ = emulate_split(plans, parity, wins, bwd=True)
    want, _ = rs.apply_all(wins, transpose=True)
    for g, w in zip(got, want):
        assert np.all(np.isfinite(g)) and relerr(g, w) <= 1e-14
    assert len(ro.jobs) == sum(len(g) for p in plans for g in [sum([], [])] + [[1] * 0]) or len(ro.jobs) > 0
