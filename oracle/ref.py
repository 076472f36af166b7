"""ctypes bindings for oracle/_ref/libbfly_ref.so — TEST INFRASTRUCTURE.

The library is the UNMODIFIED reference core (/root/reference/proj/src/*.cpp)
compiled against oracle/eigen_shim by oracle/Makefile.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may use it; the
product (``paper_0910_5435_b200``) never imports this module.

Every wrapper names the reference function it reaches.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libbfly_ref.so")
REF_ROOT = "/root/reference/proj"

_lib = None


class RefError(RuntimeError):
    pass


class RefInvalidArgument(RefError, ValueError):
    """std::invalid_argument thrown by the reference."""


def build(force: bool = False) -> str:
    """Compile the oracle (needs /root/reference; only done in the build container)."""
    if force or not os.path.exists(LIB_PATH):
        if not os.path.isdir(REF_ROOT):
            raise RefError("oracle/_ref/libbfly_ref.so missing and /root/reference absent")
        subprocess.run(["make", "-C", HERE, "-s"], check=True)
    return LIB_PATH


def available() -> bool:
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_ROOT)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        vp, i64, dbl, ip = C.c_void_p, C.c_int64, C.c_double, C.c_int
        dp = C.POINTER(C.c_double)
        L.bref_last_error.restype = C.c_char_p
        L.bref_chain_cols.restype = i64
        L.bref_chain_cols.argtypes = [ip, ip, ip]
        L.bref_plan_glrow.restype = vp
        L.bref_plan_glrow.argtypes = [ip, ip, ip, dbl, ip]
        L.bref_plan_dense.restype = vp
        L.bref_plan_dense.argtypes = [dp, i64, i64, dbl, ip]
        L.bref_plan_transform.restype = vp
        L.bref_plan_transform.argtypes = [ip, ip, ip, dbl, ip]
        L.bref_plan_load.restype = vp
        L.bref_plan_load.argtypes = [C.c_char_p, i64]
        L.bref_plan_save.restype = i64
        L.bref_plan_save.argtypes = [vp, C.c_char_p, i64]
        L.bref_plan_free.argtypes = [vp]
        L.bref_plan_info.argtypes = [vp, C.POINTER(i64), dp]
        L.bref_apply.restype = ip
        L.bref_apply.argtypes = [vp, ip, dp, i64, dp, i64, ip]
        L.bref_apply_len.restype = ip
        L.bref_apply_len.argtypes = [vp, ip, dp, i64, dp]
        L.bref_rule.restype = ip
        L.bref_rule.argtypes = [ip, ip, ip, dp, dp, dp]
        L.bref_dense_glrow.restype = ip
        L.bref_dense_glrow.argtypes = [ip, ip, ip, dp]
        L.bref_dense_transform.restype = ip
        L.bref_dense_transform.argtypes = [ip, ip, ip, dp, dp, dp]
        L.bref_planset_glrow.restype = vp
        L.bref_planset_glrow.argtypes = [ip, ip, ip, dbl, ip, ip]
        L.bref_planset_size.restype = i64
        L.bref_planset_size.argtypes = [vp]
        L.bref_planset_plan.restype = vp
        L.bref_planset_plan.argtypes = [vp, i64]
        L.bref_planset_free.argtypes = [vp]
        L.bref_planset_apply.restype = dbl
        L.bref_planset_apply.argtypes = [vp, ip, dp, C.POINTER(i64), dp, C.POINTER(i64),
                                         C.POINTER(C.c_int), ip]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().bref_last_error().decode()
    if rc == 1:
        raise RefInvalidArgument(msg)
    raise RefError(msg)


def _check_handle(h):
    if not h:
        msg = lib().bref_last_error().decode()
        if "epsilon" in msg or "block_width" in msg or "empty" in msg or "must be" in msg:
            raise RefInvalidArgument(msg)
        raise RefError(msg)
    return h


def chain_cols(l: int, mu: int, p: int) -> int:
    return int(lib().bref_chain_cols(l, mu, p))


class RefPlan:
    """A reference ``bfly::ButterflyPlan`` owned by the oracle library."""

    def __init__(self, handle, owner=None):
        self._h = handle
        self._owner = owner  # plans inside a RefPlanSet are borrowed

    def __del__(self):
        if getattr(self, "_owner", 1) is None and getattr(self, "_h", None):
            lib().bref_plan_free(self._h)
            self._h = None

    # -- constructors (reference build_plan via its ColumnSource plugins) --
    @classmethod
    def glrow(cls, l: int, mu: int, parity: int, eps: float, block_width: int = 60):
        return cls(_check_handle(lib().bref_plan_glrow(l, mu, parity, eps, block_width)))

    @classmethod
    def dense(cls, a: np.ndarray, eps: float, block_width: int = 60):
        a = np.asfortranarray(a, dtype=np.float64)
        return cls(_check_handle(lib().bref_plan_dense(_dp(a), a.shape[0], a.shape[1], eps,
                                                       block_width)))

    @classmethod
    def transform(cls, m: int, n: int, parity: int, eps: float, block_width: int = 60):
        return cls(_check_handle(lib().bref_plan_transform(m, n, parity, eps, block_width)))

    @classmethod
    def load(cls, blob: bytes):
        return cls(_check_handle(lib().bref_plan_load(blob, len(blob))))

    def save(self) -> bytes:
        n = lib().bref_plan_save(self._h, None, 0)
        if n < 0:
            _check(2)
        buf = C.create_string_buffer(int(n))
        lib().bref_plan_save(self._h, buf, n)
        return buf.raw

    def info(self) -> dict:
        info = (C.c_int64 * 10)()
        ks = (C.c_double * 2)()
        lib().bref_plan_info(self._h, info, ks)
        keys = ["n_rows", "n_cols", "levels", "stored_words", "m_max_words", "events",
                "root_groups", "k_max", "id_count", "block_width"]
        d = {k: int(v) for k, v in zip(keys, info)}
        d["k_avg"], d["k_sigma"] = float(ks[0]), float(ks[1])
        return d

    @property
    def shape(self):
        i = self.info()
        return i["n_rows"], i["n_cols"]

    def apply(self, v: np.ndarray, transpose: bool = False) -> np.ndarray:
        """bfly::apply (A v) or bfly::apply_transpose (A^T w); v is 1-D or (n, R)."""
        nr, nc = self.shape
        n_in, n_out = (nr, nc) if transpose else (nc, nr)
        v = np.asarray(v, dtype=np.float64)
        if v.ndim == 1:
            if v.shape[0] != n_in:
                out = np.empty(max(n_out, 1))
                vv = np.ascontiguousarray(v)
                _check(lib().bref_apply_len(self._h, int(transpose), _dp(vv), vv.shape[0],
                                            _dp(out)))
            return self.apply(v[:, None], transpose)[:, 0]
        if v.shape[0] != n_in:
            raise RefInvalidArgument(f"input rows {v.shape[0]}, expected {n_in}")
        vv = np.asfortranarray(v)
        out = np.empty((n_out, v.shape[1]), order="F")
        _check(lib().bref_apply(self._h, int(transpose), _dp(vv), n_in, _dp(out), n_out,
                                v.shape[1]))
        return out

    def apply_transpose(self, w: np.ndarray) -> np.ndarray:
        return self.apply(w, transpose=True)


class RefPlanSet:
    """All GL-row plans (mu, parity) of one bandlimit, built by the reference."""

    def __init__(self, l: int, eps: float, block_width: int = 60, mu_range=None,
                 nthreads: int | None = None):
        mu0, mu1 = mu_range if mu_range is not None else (0, 2 * l)
        nthreads = nthreads or os.cpu_count() or 1
        self.l = l
        self._h = _check_handle(lib().bref_planset_glrow(l, mu0, mu1, eps, block_width,
                                                         nthreads))
        self.keys = []
        for mu in range(mu0, mu1):
            for p in (0, 1):
                if chain_cols(l, mu, p) > 0:
                    self.keys.append((mu, p))
        assert len(self.keys) == lib().bref_planset_size(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().bref_planset_free(self._h)
            self._h = None

    def __len__(self):
        return len(self.keys)

    def plan(self, i: int) -> RefPlan:
        return RefPlan(lib().bref_planset_plan(self._h, i), owner=self)

    def apply_all(self, inputs: list[np.ndarray], transpose: bool, nthreads: int | None = None):
        """Reference apply / apply_transpose on every plan; inputs[i] is (n_in, R_i)."""
        nthreads = nthreads or os.cpu_count() or 1
        n = len(self.keys)
        in_off = np.zeros(n, np.int64)
        out_off = np.zeros(n, np.int64)
        nrhs = np.zeros(n, np.int32)
        l = self.l
        tot_in = tot_out = 0
        for i, (mu, p) in enumerate(self.keys):
            nc = chain_cols(l, mu, p)
            n_in, n_out = (l, nc) if transpose else (nc, l)
            x = inputs[i]
            assert x.shape[0] == n_in
            in_off[i], out_off[i], nrhs[i] = tot_in, tot_out, x.shape[1]
            tot_in += n_in * x.shape[1]
            tot_out += n_out * x.shape[1]
        flat_in = np.empty(tot_in)
        for i, x in enumerate(inputs):
            flat_in[in_off[i]:in_off[i] + x.size] = np.asfortranarray(x).ravel(order="F")
        flat_out = np.empty(tot_out)
        secs = lib().bref_planset_apply(
            self._h, int(transpose), _dp(flat_in), in_off.ctypes.data_as(C.POINTER(C.c_int64)),
            _dp(flat_out), out_off.ctypes.data_as(C.POINTER(C.c_int64)),
            nrhs.ctypes.data_as(C.POINTER(C.c_int)), nthreads)
        if secs < 0:
            _check(2)
        outs = []
        for i, (mu, p) in enumerate(self.keys):
            nc = chain_cols(l, mu, p)
            n_out = nc if transpose else l
            r = int(nrhs[i])
            outs.append(flat_out[out_off[i]:out_off[i] + n_out * r].reshape((n_out, r), order="F"))
        return outs, secs


def rule(m: int, n: int, parity: int):
    """quadrature::build_rule(m, n, parity): (nodes, weights, center_weight)."""
    nodes = np.empty(n)
    w = np.empty(n)
    c = C.c_double(0.0)
    _check(lib().bref_rule(m, n, parity, _dp(nodes), _dp(w), C.byref(c)))
    return nodes, w, c.value


def dense_glrow(l: int, mu: int, parity: int) -> np.ndarray:
    """Dense l x n_p(mu) matrix sqrt(rho_i) Pbar^mu_{mu+2j+p}(x_i) from the reference source."""
    nc = chain_cols(l, mu, parity)
    a = np.empty((l, nc), order="F")
    _check(lib().bref_dense_glrow(l, mu, parity, _dp(a)))
    return a


def dense_transform(m: int, n: int, parity: int):
    a = np.empty((n, n), order="F")
    nodes = np.empty(n)
    w = np.empty(n)
    _check(lib().bref_dense_transform(m, n, parity, _dp(a), _dp(nodes), _dp(w)))
    return a, nodes, w


class CounterRng:
    """Restatement of include/bfly/rng.hpp:12-46 (SplitMix64 over seed + counter)."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.seed = seed & self.M
        self.counter = 0

    def next_u64(self) -> int:
        self.counter += 1
        z = (self.seed + 0x9E3779B97F4A7C15 * self.counter) & self.M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def next_open(self) -> float:
        u = ((self.next_u64() >> 11) + 0.5) * 2.0 ** -53
        return 2.0 * u - 1.0

    def vector(self, n: int) -> np.ndarray:
        return np.array([self.next_open() for _ in range(n)])

    def unit_vector(self, n: int) -> np.ndarray:
        v = self.vector(n)
        nrm = np.sqrt(np.sum(v * v))
        return v / nrm if nrm > 0 else v
