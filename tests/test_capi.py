"""The C-ABI boundary and the host side of the product (no GPU needed).

* libbfly_b200.so loads and exports every function include/bfly_b200.h
  declares (and _lib.SIGNATURES binds exactly that set);
* argument errors come back as BFLY_EINVAL / BFLY_ESERIAL with the
  reference's messages (std::invalid_argument / SerializationError);
* BFLY1 plans written by the reference parse and re-serialise byte for byte;
* the product's own plan builder (paper_0910_5435_b200/csrc/builder.cpp)
  reproduces the reference builder's plan structure, and its plans match the
  reference dense matrix to the build tolerance (checked on the CPU through
  the engine emulator, tests/engine_emulator.py).
No compute call needs a device here.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_0910_5435_b200 as bb
from paper_0910_5435_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bfly_b200.h")
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    return sorted(set(re.findall(r"\b(bfly_[a-z0-9_]+)\s*\(", text)))


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def test_header_symbols_exported():
    names = declared_functions()
    assert len(names) >= 30
    raw = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(raw, n)]
    assert not missing, missing
    assert sorted(_lib.SIGNATURES) == names  # the Python binding covers exactly the header


def test_version_and_error_codes():
    L = _lib.lib()
    assert L.bfly_version().decode().startswith("bfly_b200")
    out = C.c_void_p()
    rc = L.bfly_plan_build_glrow(0, 0, 0, 1e-12, 60, C.byref(out))
    assert rc == _lib.BFLY_EINVAL and not out.value
    assert L.bfly_last_error().decode()


def test_builder_argument_errors():
    """reference tests/test_butterfly.cpp:151-154: eps <= 0 and block width 1 are rejected."""
    a = np.eye(16)
    for eps, c in ((0.0, 8), (-1.0, 8), (1e-10, 1)):
        with pytest.raises(bb.BflyInvalidArgument):
            bb.build_plan(a, eps, c)


def test_bfly1_garbage_rejected():
    with pytest.raises(bb.BflySerializationError):
        bb.ButterflyPlan.from_bfly1(b"BFLY1" + b"\0" * 7)
    blob = open(os.path.join(GOLD, "plan_glrow_l32_mu3_p1.bfly1"), "rb").read()
    with pytest.raises(bb.BflySerializationError):
        bb.ButterflyPlan.from_bfly1(blob[:-9])


def test_bfly1_round_trip_golden():
    blob = open(os.path.join(GOLD, "plan_glrow_l32_mu3_p1.bfly1"), "rb").read()
    p = bb.ButterflyPlan.from_bfly1(blob)
    assert p.to_bfly1() == blob
    assert (p.n_rows, p.n_cols) == (32, bb.chain_cols(32, 3, 1))


def test_plan_stats_match_reference(oracle):
    for mu, par in ((0, 0), (9, 1), (100, 0)):
        rp = oracle.RefPlan.glrow(64, mu, par, 1e-12)
        mine = bb.plan_stats(bb.ButterflyPlan.from_bfly1(rp.save()))
        ri = rp.info()
        assert mine.stored_words == ri["stored_words"]
        assert mine.k_max == ri["k_max"]


@pytest.mark.parametrize("l,mu,par", [(32, 0, 0), (32, 3, 1), (64, 0, 1), (64, 21, 0), (96, 150, 1)])
def test_own_builder_matches_reference_structure(oracle, l, mu, par):
    """Same ranks, pivots and layout as the reference builder (BFLY1 size and
    index bytes); values within the build tolerance of the reference dense matrix."""
    from engine_emulator import emulate
    ref_blob = oracle.RefPlan.glrow(l, mu, par, 1e-12).save()
    mine = bb.build_glrow_plan(l, mu, par, 1e-12)
    assert len(mine.to_bfly1()) == len(ref_blob)
    ri = oracle.RefPlan.load(ref_blob).info()
    mi = mine.info()
    for k in ("stored_words", "k_max", "id_count", "levels", "events", "root_groups"):
        assert mi[k] == ri[k], k
    a = oracle.dense_glrow(l, mu, par)
    x = np.random.default_rng(l + mu).standard_normal((a.shape[1], 4))
    w = np.random.default_rng(l + 2 * mu + 1).standard_normal((a.shape[0], 4))
    got, _ = emulate([mine], [x], bwd=False)
    assert relerr(got[0], a @ x) <= 1e-12
    got, _ = emulate([mine], [w], bwd=True)
    assert relerr(got[0], a.T @ w) <= 1e-12


def test_gl_rule_matches_reference(oracle):
    g = np.load(os.path.join(GOLD, "rule_l32.npz"))
    nodes, rho = np.empty(32), np.empty(32)
    _lib.check(_lib.lib().bfly_gl_rule(32, _lib.dptr(nodes), _lib.dptr(rho)))
    assert np.max(np.abs(nodes - g["nodes"])) <= 1e-15
    # the reference's weights differ from numpy's leggauss by up to ~1e-12
    # relative (src/quadrature.cpp); the product's rule sits within 1e-14 absolute
    assert np.max(np.abs(rho - g["rho"]) / g["rho"]) <= 2e-12
    x, wg = np.polynomial.legendre.leggauss(64)
    assert np.max(np.abs(rho - 2 * wg[32:])) <= 1e-14


def test_glrow_planset_order_and_shapes():
    l = 8
    plans = bb.build_glrow_planset(l, 1e-12, threads=2)
    keys = [(mu, p) for mu in range(2 * l) for p in (0, 1) if bb.chain_cols(l, mu, p) > 0]
    assert len(plans) == len(keys) == 4 * l - 1
    for pl, (mu, p) in zip(plans, keys):
        assert (pl.n_rows, pl.n_cols) == (l, bb.chain_cols(l, mu, p))


def test_coefficient_layout():
    l = 5
    offs = [bb.coeff_offset(l, m) for m in [0] + [s * mu for mu in range(1, 2 * l) for s in (1, -1)]]
    sizes = [2 * l] + [2 * l - mu for mu in range(1, 2 * l) for _ in (1, -1)]
    assert offs == list(np.cumsum([0] + sizes[:-1]))
    assert offs[-1] + sizes[-1] == 4 * l * l
    dense = np.random.default_rng(0).standard_normal((2 * l, 4 * l - 1)) + 0j
    packed = bb.pack_dense(l, dense)
    back = bb.unpack_dense(l, packed)
    assert np.array_equal(bb.pack_dense(l, back), packed)


def test_product_fails_loudly_without_library(tmp_path):
    """No CPU fallback: a missing library is an ImportError, not a silent path."""
    import subprocess
    import sys
    code = ("import os; os.environ['BFLY_LIB']=%r\n"
            "import paper_0910_5435_b200._lib as L\n"
            "try:\n    L.lib()\nexcept ImportError as e:\n    print('ok', e)\n") % str(tmp_path / "missing.so")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert out.stdout.startswith("ok"), out.stderr
