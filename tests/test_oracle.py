"""Pins of the CPU oracle (no GPU): the compiled reference and the SHT glue.

The oracle (oracle/_ref/libbfly_ref.so: the reference's own src/*.cpp built
unmodified against a from-scratch Eigen subset; oracle/sht_oracle.py: the
phi-DFT / parity glue around it) is only trusted after it reproduces the
reference's known answers and an independent dense SHT.
"""
import os

import numpy as np
import pytest

from oracle import sht_oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# -- quadrature (reference tests/test_quadrature.cpp:58-79, :160-168) ---------

def test_single_even_node_closed_form(oracle):
    nodes, w, _ = oracle.rule(0, 1, 0)
    assert abs(nodes[0] - 1 / np.sqrt(3)) <= 1e-15
    assert abs(w[0] - 2.0) <= 2e-14


def test_single_odd_node_closed_form(oracle):
    nodes, w, c = oracle.rule(0, 1, 1)
    assert abs(nodes[0] - np.sqrt(3 / 5)) <= 1e-15
    assert abs(c - 8 / 9) <= 1e-14 and abs(w[0] - 10 / 9) <= 1e-14


@pytest.mark.parametrize("n", [8, 32, 256])
def test_m0_nodes_are_gauss_legendre(oracle, n):
    nodes, w, _ = oracle.rule(0, n, 0)
    x, wg = np.polynomial.legendre.leggauss(2 * n)
    assert np.max(np.abs(nodes - x[n:])) <= 1e-13
    assert np.max(np.abs(w - 2 * wg[n:])) <= 1e-13  # rho = 2 w_GL


def test_rule_golden(oracle):
    g = np.load(os.path.join(GOLD, "rule_l32.npz"))
    nodes, rho, _ = oracle.rule(0, 32, 0)
    assert np.array_equal(nodes, g["nodes"]) and np.array_equal(rho, g["rho"])


# -- butterfly apply (reference tests/test_butterfly.cpp:48-61, :135-155) -----

def test_identity_plan(oracle):
    p = oracle.RefPlan.dense(np.eye(256), 1e-14, 60)
    v = oracle.CounterRng(17).unit_vector(256)
    assert np.max(np.abs(p.apply(v) - v)) <= 1e-13
    assert np.max(np.abs(p.apply_transpose(v) - v)) <= 1e-13
    assert p.info()["k_max"] == 60


def kernel_matrix(n):
    i = np.arange(n)[:, None] + 0.5
    j = np.arange(n)[None, :] + 0.5
    return np.cos(8.0 * np.pi * i * j / n) / np.sqrt(n)


def test_zero_maps_to_zero_and_length_errors(oracle):
    p = oracle.RefPlan.dense(kernel_matrix(64), 1e-13, 16)
    assert np.max(np.abs(p.apply(np.zeros(64)))) == 0.0
    assert np.max(np.abs(p.apply_transpose(np.zeros(64)))) == 0.0
    with pytest.raises(oracle.RefInvalidArgument):
        p.apply(np.zeros(63))
    with pytest.raises(oracle.RefInvalidArgument):
        p.apply_transpose(np.zeros(65))


def test_dense_plan_against_dense(oracle):
    a = kernel_matrix(300)
    p = oracle.RefPlan.dense(a, 1e-13, 60)
    x = np.random.default_rng(3).standard_normal((300, 3))
    assert relerr(p.apply(x), a @ x) <= 1e-12
    assert relerr(p.apply_transpose(x), a.T @ x) <= 1e-12


def test_save_load_bit_identical(oracle):
    p = oracle.RefPlan.glrow(64, 5, 0, 1e-12)
    q = oracle.RefPlan.load(p.save())
    x = np.random.default_rng(5).standard_normal((p.shape[1], 2))
    assert np.array_equal(p.apply(x), q.apply(x))
    assert q.save() == p.save()


# -- transform plans (reference tests/test_transform.cpp:23-42, test_cli.cpp:93-123)

def test_tiny_transform_columns(oracle):
    p = oracle.RefPlan.transform(0, 4, 0, 1e-14)
    a, _, _ = oracle.dense_transform(0, 4, 0)
    for j in range(4):
        e = np.zeros(4)
        e[j] = 1.0
        assert np.max(np.abs(p.apply(e) - a[:, j])) <= 1e-13


@pytest.mark.parametrize("parity", [0, 1])
def test_size_one_transform_is_a_sign(oracle, parity):
    p = oracle.RefPlan.transform(0, 1, parity, 1e-14)
    assert abs(abs(p.apply(np.ones(1))[0]) - 1.0) <= 1e-12


def test_transform_column17_golden(oracle):
    g = np.load(os.path.join(GOLD, "transform_m3_n64.npz"))
    p = oracle.RefPlan.transform(3, 64, 0, 1e-12)
    e = np.zeros(64)
    e[17] = 1.0
    col = p.apply(e)
    assert np.array_equal(col, g["col17"])
    assert np.max(np.abs(col - g["dense_col17"])) <= 1e-12


def test_glrow_plan_golden(oracle):
    g = np.load(os.path.join(GOLD, "plan_glrow_l32_mu3_p1.npz"))
    blob = open(os.path.join(GOLD, "plan_glrow_l32_mu3_p1.bfly1"), "rb").read()
    p = oracle.RefPlan.glrow(32, 3, 1, 1e-12)
    assert p.save() == blob
    assert np.array_equal(p.apply(g["x"]), g["ax"])
    assert np.array_equal(p.apply_transpose(g["w"]), g["atw"])
    assert relerr(g["ax"], g["dense"] @ g["x"]) <= 1e-12


def test_glrow_columns_orthonormal(oracle):
    """Lemma 4 of the paper: the l-node rule integrates every same-chain product exactly."""
    for mu, p in ((0, 0), (7, 1), (40, 0)):
        a = oracle.dense_glrow(32, mu, p)
        assert np.max(np.abs(a.T @ a - np.eye(a.shape[1]))) <= 1e-13


# -- SHT glue -------------------------------------------------------------------

@pytest.mark.parametrize("l", [4, 8, 12])
def test_ref_sht_against_dense_scipy(oracle, l):
    from oracle.sht_oracle import RefSHT, dense_synthesis, random_coefficients
    sht = RefSHT(l, 1e-13)
    beta = random_coefficients(l, 1, 11 + l)
    grid = sht.synthesize(beta)
    want = dense_synthesis(l, beta[0], sht.cos_theta())
    assert relerr(grid[0], want) <= 1e-12
    assert relerr(sht.analyze(grid), beta) <= 1e-12


@pytest.mark.parametrize("l", [16, 32])
def test_ref_sht_golden(oracle, l):
    from oracle.sht_oracle import RefSHT, random_coefficients
    g = np.load(os.path.join(GOLD, f"sht_l{l}.npz"))
    beta = random_coefficients(l, 2, int(g["seed"]), decaying_member=1)
    assert np.array_equal(beta, g["beta"])
    sht = RefSHT(l, float(g["eps"]))
    grid = sht.synthesize(beta)
    assert relerr(grid, g["grid"]) <= 1e-14
    assert relerr(sht.analyze(g["grid"]), g["back"]) <= 1e-14
    assert relerr(g["back"], beta) <= 1e-11


def test_counter_rng_is_splitmix(oracle):
    """include/bfly/rng.hpp: outputs in (-1, 1), deterministic per seed."""
    a = oracle.CounterRng(17).vector(1000)
    b = oracle.CounterRng(17).vector(1000)
    assert np.array_equal(a, b) and np.all(np.abs(a) < 1) and abs(a.mean()) < 0.1


def test_pbar_rows_matches_independent_dense():
    """The extended-precision recurrence against scipy's lpmv route (small l)."""
    l = 6
    x = np.linspace(-0.95, 0.95, 7)
    for mu in (0, 1, 3):
        beta = np.zeros((1, 4 * l * l), dtype=np.complex128)
        o = sht_oracle.coeff_offset(l, mu)
        beta[0, o:o + 2 * l - mu] = np.arange(1, 2 * l - mu + 1)
        f = sht_oracle.dense_synthesis(l, beta, x)[0, :, 0]  # phi = 0
        mine = (np.arange(1, 2 * l - mu + 1)[:, None] * sht_oracle.pbar_rows_extended(l, mu, x)).sum(axis=0).astype(np.float64)
        assert np.allclose(mine, f.real, rtol=1e-13, atol=1e-13)
