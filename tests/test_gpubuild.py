"""GPU plan construction (csrc/gpubuild.cu) against the reference.

The plans come out of the batched cluster IDs; what is checked is what makes
them the reference's kind of plan: the BFLY1 structure round trips, every plan
applies (forward and transpose, numpy emulator of the device program) within
its ID precision of the reference's dense matrix (src/transform.cpp:37-60 on
build_rule(0, l, even)), and the compression (stored words, ranks, levels) is
that of the host builder / reference policy (src/butterfly.cpp:194-382) up to
pivot ties.
"""
import numpy as np
import pytest

import paper_0910_5435_b200 as bb

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _keys(l):
    return [(mu, p) for mu in range(2 * l) for p in (0, 1) if bb.chain_cols(l, mu, p) > 0]


@pytest.mark.parametrize("l,eps", [(1, 1e-12), (2, 1e-12), (5, 1e-12), (32, 1e-12), (96, 1e-12), (256, 1e-12),
                                   (256, 1e-10)])
def test_gpu_plans_vs_reference_dense(oracle, l, eps, monkeypatch):
    from engine_emulator import emulate
    nodes, rho, _ = oracle.rule(0, l, 0)
    monkeypatch.setenv("BFLY_BUILDER", "gpu")
    gpu = bb.build_glrow_planset(l, eps, rule=(nodes, rho))
    monkeypatch.setenv("BFLY_BUILDER", "host")
    host = bb.build_glrow_planset(l, eps, rule=(nodes, rho), threads=8)
    keys = _keys(l)
    assert len(gpu) == len(host) == len(keys)
    sw_g = sum(p.info()["stored_words"] for p in gpu)
    sw_h = sum(p.info()["stored_words"] for p in host)
    assert abs(sw_g - sw_h) <= 0.02 * sw_h + 64, (sw_g, sw_h)
    rng = np.random.default_rng(l)
    sample = range(len(keys)) if len(keys) <= 48 else sorted(rng.choice(len(keys), 48, replace=False))
    for i in sample:
        mu, p = keys[i]
        gp, hp = gpu[i], host[i]
        gi, hi = gp.info(), hp.info()
        assert (gi["n_rows"], gi["n_cols"]) == (l, bb.chain_cols(l, mu, p))
        assert abs(gi["levels"] - hi["levels"]) <= 1, (mu, p, gi, hi)
        # BFLY1 structure: serialise, parse, same bytes
        blob = gp.to_bfly1()
        assert bb.ButterflyPlan.from_bfly1(blob).to_bfly1() == blob
        a = oracle.dense_glrow(l, mu, p)
        x = rng.standard_normal((a.shape[1], 4))
        w = rng.standard_normal((a.shape[0], 4))
        got, _ = emulate([gp], [x], bwd=False)
        assert relerr(got[0], a @ x) <= 20 * eps, (mu, p)
        got, _ = emulate([gp], [w], bwd=True)
        assert relerr(got[0], a.T @ w) <= 20 * eps, (mu, p)


def test_gpu_plans_match_reference_structure(oracle, monkeypatch):
    """Ranks and levels of the reference builder on its own grid (pivots may
    differ on near-ties: the norms here are exact, the reference downdates)."""
    l = 128
    nodes, rho, _ = oracle.rule(0, l, 0)
    monkeypatch.setenv("BFLY_BUILDER", "gpu")
    gpu = bb.build_glrow_planset(l, 1e-12, rule=(nodes, rho))
    keys = _keys(l)
    diffs = []
    for i in range(0, len(keys), 9):
        mu, p = keys[i]
        ri = oracle.RefPlan.glrow(l, mu, p, 1e-12).info()
        gi = gpu[i].info()
        assert gi["levels"] == ri["levels"] and gi["events"] == ri["events"], (mu, p, gi, ri)
        diffs.append(abs(gi["stored_words"] - ri["stored_words"]) / ri["stored_words"])
    assert max(diffs) <= 0.03, diffs


def test_gpu_builder_sht_vs_oracle(oracle, monkeypatch):
    """The default (GPU-built) plans in the full transform, on the reference grid."""
    import torch
    from oracle import sht_oracle
    monkeypatch.setenv("BFLY_BUILDER", "gpu")
    l, B = 256, 3
    ref = sht_oracle.RefSHT(l, 1e-12)
    sht = bb.SHT(l, eps=1e-12, rule=(ref.nodes, ref.rho))
    beta = sht_oracle.random_coefficients(l, B, seed=77)
    g_ref = ref.synthesize(beta)
    grid = sht.synthesize(torch.from_numpy(beta).cuda()).cpu().numpy()
    assert relerr(grid, g_ref) <= 1e-10
    back = sht.analyze(torch.from_numpy(g_ref).cuda()).cpu().numpy()
    assert relerr(back, ref.analyze(g_ref)) <= 1e-10
