"""Parity of the CUDA butterfly engine with the reference CPU apply.

The same reference-built plan (bfly::build_plan, moved across the boundary as
its BFLY1 bytes) is applied by the reference (bfly::apply / apply_transpose,
src/butterfly.cpp:384-513, one vector per call) and by the engine (all
right-hand sides in one launch).  Matrices follow the reference's own tests
(tests/test_butterfly.cpp, tests/test_transform.cpp).  Tolerance: relative l2
<= 1e-13 for identical plans (fp64 summation order is the only difference).
"""
import numpy as np
import pytest

import paper_0910_5435_b200 as bb

pytestmark = pytest.mark.gpu
TOL_SAME_PLAN = 1e-13


def kernel_matrix(n):
    i = np.arange(n)[:, None] + 0.5
    j = np.arange(n)[None, :] + 0.5
    return np.cos(8.0 * np.pi * i * j / n) / np.sqrt(n)


def low_rank(n, rank, seed):
    from oracle.ref import CounterRng
    rng = CounterRng(seed)
    u = np.empty((n, rank))
    w = np.empty((rank, n))
    for a in range(n):
        for b in range(rank):
            u[a, b] = rng.next_open()
            w[b, a] = rng.next_open()
    return u @ w / n


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


CASES = {
    "identity256": lambda: (np.eye(256), 1e-14, 60),
    "lowrank480": lambda: (low_rank(480, 10, 3), 1e-12, 60),
    "kernel300": lambda: (kernel_matrix(300), 1e-13, 60),
    "ragged130": lambda: (kernel_matrix(130), 1e-13, 60),
    "kernel64_c16": lambda: (kernel_matrix(64), 1e-13, 16),
    "narrow40x7": lambda: (np.random.default_rng(71).uniform(-1, 1, (40, 7)), 1e-13, 60),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("nrhs", [1, 3, 4, 9, 16, 70, 300])
def test_dense_sources_match_reference(oracle, name, nrhs):
    """nrhs >= 16 runs the wave programs (FP64 tensor cores), 70 = two 64-column chunks,
    300 = two passes of at most 256 right-hand sides."""
    a, eps, c = CASES[name]()
    rp = oracle.RefPlan.dense(a, eps, c)
    plan = bb.ButterflyPlan.from_bfly1(rp.save())
    rng = np.random.default_rng(nrhs)
    v = rng.standard_normal((a.shape[1], nrhs))
    w = rng.standard_normal((a.shape[0], nrhs))
    assert relerr(bb.apply(plan, v), rp.apply(v)) <= TOL_SAME_PLAN
    assert relerr(bb.apply_transpose(plan, w), rp.apply_transpose(w)) <= TOL_SAME_PLAN
    # and the plan still represents the matrix (reference tests/test_butterfly.cpp:33-44)
    assert np.max(np.abs(bb.apply(plan, v) - a @ v)) <= 1e-10 * max(1.0, np.abs(a @ v).max())


def test_reference_transform_plans(oracle):
    # tests/test_transform.cpp:67-82 (m=64, n=512, odd) and :54-65 (m=0, n=512, even)
    for m, n, par in [(64, 512, 1), (0, 512, 0), (3, 256, 1)]:
        rp = oracle.RefPlan.transform(m, n, par, 1e-14)
        plan = bb.ButterflyPlan.from_bfly1(rp.save())
        v = np.random.default_rng(m).standard_normal((n, 5))
        assert relerr(bb.forward(plan, v), rp.apply(v)) <= TOL_SAME_PLAN
        assert relerr(bb.inverse(plan, v), rp.apply_transpose(v)) <= TOL_SAME_PLAN
        back = bb.inverse(plan, bb.forward(plan, v))
        assert np.max(np.abs(back - v)) <= 1e-10 * np.abs(v).max()


def test_zero_maps_to_exact_zero(oracle):
    rp = oracle.RefPlan.dense(kernel_matrix(64), 1e-13, 16)
    plan = bb.ButterflyPlan.from_bfly1(rp.save())
    assert np.all(bb.apply(plan, np.zeros(64)) == 0.0)
    assert np.all(bb.apply_transpose(plan, np.zeros(64)) == 0.0)


def test_length_errors_follow_reference():
    plan = bb.build_plan(kernel_matrix(64), 1e-13, 16)
    with pytest.raises(ValueError, match="apply: vector length 63, expected 64"):
        bb.apply(plan, np.zeros(63))
    with pytest.raises(ValueError, match="apply_transpose: vector length 65, expected 64"):
        bb.apply_transpose(plan, np.zeros(65))


def test_adjoint_identity():
    plan = bb.build_plan(kernel_matrix(300), 1e-13, 60)
    rng = np.random.default_rng(43)
    v = rng.standard_normal((300, 10))
    w = rng.standard_normal((300, 10))
    lhs = np.sum(bb.apply(plan, v) * w, axis=0)
    rhs = np.sum(v * bb.apply_transpose(plan, w), axis=0)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.abs(lhs).max()


def test_torch_device_path_matches_host_path():
    import torch
    plan = bb.build_plan(kernel_matrix(300), 1e-13, 60)
    v = np.random.default_rng(5).standard_normal((300, 7))
    host = bb.apply(plan, v)
    dev = bb.apply(plan, torch.from_numpy(v).cuda()).cpu().numpy()
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("l,nrhs", [(32, 4), (256, 4), (32, 19), (256, 40)])
def test_glrow_planset_one_launch(oracle, l, nrhs):
    """Every (mu, parity) plan of a bandlimit in ONE apply vs the reference: the
    engine (4 right-hand sides) or the wave programs (19, 40)."""
    rs = oracle.RefPlanSet(l, 1e-12)
    plans = [bb.ButterflyPlan.from_bfly1(rs.plan(i).save()) for i in range(len(rs))]
    ps = bb.PlanSet(plans)
    rng = np.random.default_rng(l)
    ins = [rng.standard_normal((p.n_cols, nrhs)) for p in plans]
    flat, _ = ps.stack(ins)
    got = ps.unstack(ps.apply_host(flat, nrhs, False), nrhs, False)
    want, _ = rs.apply_all(ins, transpose=False)
    for g, w in zip(got, want):
        assert relerr(g, w) <= TOL_SAME_PLAN
    wins = [rng.standard_normal((l, nrhs)) for _ in plans]
    flat, _ = ps.stack(wins)
    got = ps.unstack(ps.apply_host(flat, nrhs, True), nrhs, True)
    want, _ = rs.apply_all(wins, transpose=True)
    for g, w in zip(got, want):
        assert relerr(g, w) <= TOL_SAME_PLAN


def test_bench_rows_gpu_mode(tmp_path, capsys):
    """GPU `bfly bench` rows (reference CSV schema, tools/bfly_main.cpp:166-183) for a
    reference-built BFLY1 plan: the schema, the plan statistics, positive device
    times and the round-trip column (orthonormal GL-row columns: A^T A = I)."""
    import os
    from paper_0910_5435_b200 import bench_rows
    path = os.path.join(os.path.dirname(__file__), "golden", "plan_glrow_l32_mu3_p1.bfly1")
    assert bench_rows.main([path, "--m", "3", "--parity", "odd"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == bench_rows.HEADER
    row = dict(zip(lines[0].split(","), lines[1].split(",")))
    with open(path, "rb") as f:
        info = bb.ButterflyPlan.from_bfly1(f.read()).info()
    assert row["n"] == str(info["n_cols"]) and row["m"] == "3" and row["parity"] == "odd"
    assert row["k_max"] == str(info["k_max"]) and row["m_max"] == str(info["m_max_words"])
    assert float(row["t_fwd"]) > 0 and float(row["t_inv"]) > 0
    assert float(row["eps_inv"]) <= 1e-12
    assert row["t_dir"] == "NA" and row["eps_fwd"] == "NA"
