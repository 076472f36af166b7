"""Oracle parity at BASELINE.json's large configurations (c3 in full, c4 and
l = 4096 on sampled order ranges).

The oracle is the reference's own bfly::apply / apply_transpose
(/root/reference/proj/src/butterfly.cpp:384-513, compiled unmodified into
oracle/_ref) on reference-built GL-row plans, plus the restated parity
combine / phi DFT of oracle/sht_oracle.py.  Two bars (north_star: relative
l2 <= 1e-10 in fp64 at ID precision 1e-12):

* this library's own plans: <= 1e-10;
* the reference's plans moved across the boundary as BFLY1 bytes, with the
  reference's weights (so only the apply path differs): <= 1e-12.

The grid is the quadrature's: the reference's build_rule(0, l, even) carries
node errors up to ~2e-14 near the equator and weight errors up to ~2e-8
(relative) next to the poles at l = 2048 (mpmath check), which
moves P(x_i) by ~1e-9 relative at l = 4096; this library's own rule is within
~6e-17 / ~7e-11.  So the order-range cases build this library's plans on the
reference's rule (SHT.range(rule=...)) — what a drop-in caller holding the
reference's TransformPlan grid gets — and test_own_rule_accuracy holds the
default rule's transform against an independent extended-precision dense
evaluation.

c3 (l = 1024, 16 functions, member 15 with a (k+1)^-2 spectrum) runs in full:
both directions, on the wave programs (the batch) and on the whole-chain
engine (single functions).  At l = 2048 (c4, 64 functions, eps 1e-12 and
1e-10) and l = 4096 (c5, 8 functions) the full-size oracle would take
CPU-hours, so sampled order ranges — the lowest orders (mu = 0 has R = 2B),
the middle and the top (the near-empty chains at mu = 2l - 1) — run through
the same entry points the order-sharded transform uses (SHT.range), with the
whole batch, so R = 4B right-hand sides (256 at c4: four 64-column chunks)
go through every DMMA tile path.
"""
import numpy as np
import pytest
import torch

import paper_0910_5435_b200 as bb
from oracle import sht_oracle
from paper_0910_5435_b200.sharded import coefficient_slices

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# --------------------------------------------------------------------------- c3
@pytest.fixture(scope="module")
def c3(oracle):
    l, B = 1024, 16
    ref = sht_oracle.RefSHT(l, 1e-12)
    beta = sht_oracle.random_coefficients(l, B, seed=1003, decaying_member=B - 1)
    g_ref = ref.synthesize(beta)
    back_ref = ref.analyze(g_ref)
    return l, B, ref, beta, g_ref, back_ref


def _c3_check(sht, beta, g_ref, back_ref, tol):
    B = beta.shape[0]
    assert sht.uses_waves(B)
    tb = torch.from_numpy(beta).cuda()
    grid = sht.synthesize(tb)
    errs = {"synth_waves": relerr(grid.cpu().numpy(), g_ref)}
    tg = torch.from_numpy(g_ref).cuda()
    errs["anal_waves"] = relerr(sht.analyze(tg).cpu().numpy(), back_ref)
    # the decaying member on its own (tiny norm next to the i.i.d. members)
    d = B - 1
    errs["anal_waves_decaying"] = relerr(sht.analyze(tg[d:d + 1]).cpu().numpy()[0], back_ref[d])
    # single functions run on the whole-chain engine
    for b in (0, d):
        assert not sht.uses_waves(1)
        errs[f"synth_engine_{b}"] = relerr(sht.synthesize(tb[b:b + 1]).cpu().numpy()[0], g_ref[b])
        errs[f"anal_engine_{b}"] = relerr(sht.analyze(tg[b:b + 1]).cpu().numpy()[0], back_ref[b])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, (errs, tol)
    return errs


def test_c3_own_plans_vs_oracle(c3):
    l, B, ref, beta, g_ref, back_ref = c3
    sht = bb.SHT(l, eps=1e-12)
    _c3_check(sht, beta, g_ref, back_ref, 1e-10)


def test_c3_reference_plans_vs_oracle(c3):
    """The reference's own 4095 plans (BFLY1 bytes) and GL weights: only the
    apply path differs from the oracle."""
    l, B, ref, beta, g_ref, back_ref = c3
    plans = [bb.ButterflyPlan.from_bfly1(ref.plans.plan(i).save()) for i in range(len(ref.plans))]
    sht = bb.SHT.from_plans(l, plans, rho=ref.rho)
    _c3_check(sht, beta, g_ref, back_ref, 1e-12)


# ---------------------------------------------------------- c4 / c5 order ranges
def _range_case(oracle, l, B, eps, mu0, mu1, seed):
    """One sampled order range at full batch: own plans (<= 1e-10) and the
    reference plans (<= 1e-12), synthesis and analysis."""
    rs = oracle.RefPlanSet(l, eps, mu_range=(mu0, mu1))
    ref = sht_oracle.RefSHT(l, eps, planset=rs)
    bins = ref.range_bins()
    N = 4 * l - 1
    rng = np.random.default_rng(seed)
    slices = coefficient_slices(l, mu0, mu1)
    # host coefficients: np.zeros is lazily allocated, only the range's slices
    # are touched (17 GB at l = 2048, B = 64 would not be written out)
    beta = np.zeros((B, 4 * l * l), dtype=np.complex128)
    for a, b in slices:
        beta[:, a:b] = rng.standard_normal((B, b - a)) + 1j * rng.standard_normal((B, b - a))
    g_ref = ref.legendre_synthesis_bins(beta)                  # (B, 2l, nbins)
    gin = rng.standard_normal(g_ref.shape) + 1j * rng.standard_normal(g_ref.shape)
    back_ref = np.zeros((B, 4 * l * l), dtype=np.complex128)
    ref.legendre_analysis_bins(gin, back_ref)

    dev = torch.device("cuda", 0)
    beta_d = torch.zeros((B, 4 * l * l), dtype=torch.complex128, device=dev)
    for a, b in slices:
        beta_d[:, a:b] = torch.from_numpy(np.ascontiguousarray(beta[:, a:b])).to(dev)
    bins_t = torch.tensor(bins, device=dev)
    gin_d = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device=dev)
    gin_d[bins_t] = torch.from_numpy(np.ascontiguousarray(np.transpose(gin, (2, 0, 1)))).to(dev)
    want_b = np.concatenate([back_ref[:, a:b] for a, b in slices], axis=1)

    plans_ref = [bb.ButterflyPlan.from_bfly1(rs.plan(i).save()) for i in range(len(rs))]
    rule_ref = (ref.nodes, ref.rho)
    errs = {}
    # own: this library's builder on the reference's grid (its build_rule
    # nodes and weights); refplans: the reference's plans and weights
    for name, sht in (("own", bb.SHT.range(l, mu0, mu1, eps=eps, rule=rule_ref)),
                      ("refplans", bb.SHT.range(l, mu0, mu1, eps=eps, plans=plans_ref, rho=ref.rho))):
        assert sht.uses_waves(B)
        gout = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device=dev)
        sht.legendre_synthesize(beta_d, out=gout)
        got_g = gout[bins_t].permute(1, 2, 0).cpu().numpy()
        errs[f"synth_{name}"] = relerr(got_g, g_ref)
        # nothing outside the range's bins is written
        assert float(gout.abs().sum().item()) == pytest.approx(float(gout[bins_t].abs().sum().item()))
        del gout
        bout = torch.zeros((B, 4 * l * l), dtype=torch.complex128, device=dev)
        sht.legendre_analyze(gin_d, out=bout)
        got_b = torch.cat([bout[:, a:b] for a, b in slices], dim=1).cpu().numpy()
        errs[f"anal_{name}"] = relerr(got_b, want_b)
        del bout, sht
    torch.cuda.empty_cache()
    return errs


C4_RANGES = [(0, 8), (1020, 1028), (4088, 4096)]


@pytest.mark.parametrize("eps", [1e-12, 1e-10])
@pytest.mark.parametrize("mu0,mu1", C4_RANGES)
def test_c4_order_ranges_vs_oracle(oracle, eps, mu0, mu1):
    """BASELINE.json configs[3]: l = 2048, 64 functions (R = 256), eps 1e-12 and 1e-10."""
    errs = _range_case(oracle, 2048, 64, eps, mu0, mu1, seed=int(mu0 + 1e6 * eps))
    assert errs["synth_own"] <= 1e-10 and errs["anal_own"] <= 1e-10, errs
    assert errs["synth_refplans"] <= 1e-12 and errs["anal_refplans"] <= 1e-12, errs


@pytest.mark.parametrize("mu0,mu1", [(0, 4), (4094, 4098), (8188, 8192)])
def test_l4096_order_ranges_vs_oracle(oracle, mu0, mu1):
    """BASELINE.json configs[4]: l = 4096, 8 functions (R = 32), eps 1e-12."""
    errs = _range_case(oracle, 4096, 8, 1e-12, mu0, mu1, seed=4096 + mu0)
    assert errs["synth_own"] <= 1e-10 and errs["anal_own"] <= 1e-10, errs
    assert errs["synth_refplans"] <= 1e-12 and errs["anal_refplans"] <= 1e-12, errs


# ------------------------------------------------- back-to-back launches (PDL)
@pytest.mark.parametrize("l,B", [(128, 1), (128, 2), (64, 1)])
def test_back_to_back_directions_no_gap(oracle, l, B):
    """analyze -> synthesize -> analyze ... on one stream with no kernel in
    between: the engine launches chain by programmatic dependent launch and
    share one task counter per program, so a grid must not claim tasks while
    its predecessor is still claiming (1-stage first-wave jobs at l = 128)."""
    ref = sht_oracle.RefSHT(l, 1e-12)
    sht = bb.SHT(l, eps=1e-12)
    beta = sht_oracle.random_coefficients(l, B, seed=77 + l + B)
    g_ref = ref.synthesize(beta)
    tb = torch.from_numpy(beta).cuda()
    grid = sht.synthesize(tb)
    outs = []
    for _ in range(20):
        back = sht.analyze(grid)
        grid = sht.synthesize(back)
        outs.append((back, grid))
    torch.cuda.synchronize()
    for back, g in outs:
        assert relerr(back.cpu().numpy(), beta) <= 1e-10
        assert relerr(g.cpu().numpy(), g_ref) <= 1e-10


# ------------------------------------------- the default rule against truth
@pytest.mark.parametrize("l", [2048, 4096])
def test_own_rule_accuracy(l):
    """The default rule (this library's GL nodes and weights) on the lowest
    orders, where the grid's pole rows carry the largest Legendre values: the
    Legendre synthesis against Sum_k beta_k Pbar_k(x_i) evaluated in extended
    precision at the same nodes, <= 1e-10 (ID precision 1e-12 per block;
    measured 4e-11 at l = 4096 mu = 0 through six levels).  (The
    reference's rule moves the same values by ~1e-9 at l = 4096; see the
    module docstring.)"""
    mu0, mu1, B = 0, 2, 2
    sht = bb.SHT.range(l, mu0, mu1, eps=1e-12)
    nodes, _ = sht.rule()
    rng = np.random.default_rng(l)
    beta = np.zeros((B, 4 * l * l), dtype=np.complex128)
    for a, b in coefficient_slices(l, mu0, mu1):
        beta[:, a:b] = rng.standard_normal((B, b - a)) + 1j * rng.standard_normal((B, b - a))
    N = 4 * l - 1
    dev = torch.device("cuda", 0)
    gout = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device=dev)
    sht.legendre_synthesize(torch.from_numpy(beta).to(dev), out=gout)
    errs = {}
    for m in (0, 1, -1):
        mu = abs(m)
        P = sht_oracle.pbar_rows_extended(l, mu, nodes)                              # (2l - mu, l)
        sign = np.where((np.arange(mu, 2 * l) - mu) % 2 == 0, 1, -1)[:, None]
        o = sht_oracle.coeff_offset(l, m)
        c = beta[:, o:o + 2 * l - mu].astype(np.clongdouble)      # (B, 2l - mu)
        gp = (c @ P).astype(np.complex128)                        # g(+x_i)
        gm = (c @ (sign * P)).astype(np.complex128)               # g(-x_i)
        want = np.concatenate([gm[:, ::-1], gp], axis=1)          # rows t: -x_{l-1-t} then +x_{t-l}
        got = gout[m % N].cpu().numpy()
        errs[m] = relerr(got, want)
    assert max(errs.values()) <= 1e-10, errs
