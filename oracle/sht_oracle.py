"""CPU oracle for the full spherical harmonic transform — TEST INFRASTRUCTURE.

The Legendre stage is the UNMODIFIED reference (bfly::apply /
bfly::apply_transpose, /root/reference/proj/src/butterfly.cpp:384-513, via
oracle/_ref/libbfly_ref.so) on every GL-row plan, one right-hand side per
call, exactly like the reference API; threads run over plans.  The reference
has no phi stage and no +-x combine (SURVEY.md §2 "new
components"), so this module restates them from the paper:

  * grid and expansion: arXiv 0910.5435 eqs. (expansion), (thetas),
    (alternate_expansion); longitudes phi_n = 2 pi n/(4l-1)
    as BASELINE.json specifies;
  * parity split: Pbar^mu_k(-x) = (-1)^(k-mu) Pbar^mu_k(x),
    so g(+-x_i) = (u_even +- u_odd) / sqrt(rho_i) and, for analysis,
    u_p,i = sqrt(rho_i) (g(+x_i) +- g(-x_i)) / 2  (rho_i = 2 w_GL,i);
  * phi stage: numpy.fft over m in bin order (m mod 4l-1).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use it.
``dense_synthesis`` is an independent O(l^3) check with scipy's Legendre
functions (no reference code) used to pin conventions at small l.
"""
from __future__ import annotations

import numpy as np

from . import ref


def coeff_offset(l: int, m: int) -> int:
    mu = abs(m)
    base = 0 if mu == 0 else 2 * l + (mu - 1) * (4 * l - mu)
    return base + (2 * l - mu if m < 0 else 0)


def chain_rhs(l: int, beta: np.ndarray, mu: int, p: int) -> np.ndarray:
    """Right-hand sides of chain p at order mu: (n_p, R), R = (b, sign, re/im)."""
    B = beta.shape[0]
    nc = ref.chain_cols(l, mu, p)
    signs = (0,) if mu == 0 else (0, 1)
    cols = []
    for b in range(B):
        for s in signs:
            o = coeff_offset(l, mu if s == 0 else -mu)
            seg = beta[b, o + p: o + p + 2 * nc: 2]  # degrees mu + 2j + p
            cols.append(seg.real)
            cols.append(seg.imag)
    return np.stack(cols, axis=1)


def scatter_rhs(l: int, beta: np.ndarray, mu: int, p: int, x: np.ndarray) -> None:
    B = beta.shape[0]
    nc = ref.chain_cols(l, mu, p)
    signs = (0,) if mu == 0 else (0, 1)
    c = 0
    for b in range(B):
        for s in signs:
            o = coeff_offset(l, mu if s == 0 else -mu)
            beta[b, o + p: o + p + 2 * nc: 2] = x[:, c] + 1j * x[:, c + 1]
            c += 2


class RefSHT:
    """Reference-backed SHT of bandlimit l on the reference's GL-row plans."""

    def __init__(self, l: int, eps: float = 1e-12, block_width: int = 60, nthreads=None,
                 planset: ref.RefPlanSet | None = None):
        self.l = l
        self.N = 4 * l - 1
        self.plans = planset or ref.RefPlanSet(l, eps, block_width, nthreads=nthreads)
        nodes, rho, _ = ref.rule(0, l, 0)
        self.nodes, self.rho = nodes, rho
        self.nthreads = nthreads

    def cos_theta(self) -> np.ndarray:
        return np.concatenate([-self.nodes[::-1], self.nodes])

    # Legendre stage only ------------------------------------------------------
    def legendre_synthesis(self, beta: np.ndarray):
        """beta (B, 4l^2) -> g bins (B, 2l, N); returns (g, seconds in reference apply)."""
        l, N = self.l, self.N
        beta = np.atleast_2d(beta)
        B = beta.shape[0]
        ins = [chain_rhs(l, beta, mu, p) for (mu, p) in self.plans.keys]
        outs, secs = self.plans.apply_all(ins, transpose=False, nthreads=self.nthreads)
        g = np.zeros((B, 2 * l, N), dtype=np.complex128)
        u = {}
        for (mu, p), o in zip(self.plans.keys, outs):
            u[(mu, p)] = o
        isr = 1.0 / np.sqrt(self.rho)
        for mu in sorted({mu for (mu, _) in self.plans.keys}):  # all orders, or the plan set's range
            ue = u[(mu, 0)]
            uo = u.get((mu, 1), np.zeros_like(ue))
            gp = (ue + uo) * isr[:, None]
            gm = (ue - uo) * isr[:, None]
            signs = (0,) if mu == 0 else (0, 1)
            c = 0
            for b in range(B):
                for s in signs:
                    binm = mu if s == 0 else N - mu
                    g[b, l:, binm] = gp[:, c] + 1j * gp[:, c + 1]
                    g[b, :l, binm] = (gm[:, c] + 1j * gm[:, c + 1])[::-1]
                    c += 2
        return g, secs

    def legendre_analysis(self, gdft: np.ndarray):
        """Unnormalised forward DFT rows (B, 2l, N) -> beta (B, 4l^2); (beta, seconds)."""
        l, N = self.l, self.N
        gdft = np.asarray(gdft)
        B = gdft.shape[0]
        g = gdft / N
        hs = np.sqrt(self.rho) / 2.0
        ins = []
        for (mu, p) in self.plans.keys:
            signs = (0,) if mu == 0 else (0, 1)
            cols = []
            for b in range(B):
                for s in signs:
                    binm = mu if s == 0 else N - mu
                    gp = g[b, l:, binm]
                    gm = g[b, :l, binm][::-1]
                    u = (gp + gm) if p == 0 else (gp - gm)
                    u = u * hs
                    cols.append(u.real)
                    cols.append(u.imag)
            ins.append(np.stack(cols, axis=1))
        outs, secs = self.plans.apply_all(ins, transpose=True, nthreads=self.nthreads)
        beta = np.zeros((B, 4 * l * l), dtype=np.complex128)
        for (mu, p), o in zip(self.plans.keys, outs):
            scatter_rhs(l, beta, mu, p, o)
        return beta, secs

    # Legendre stage on the plan set's orders only (sampled order ranges at large l,
    # where the full (B, 2l, 4l-1) bin array would not fit host memory) --------
    def range_bins(self) -> list[int]:
        """phi bins (m mod 4l-1) of the plan set's orders, in the order the *_bins
        methods use: for each mu ascending, +mu then (mu > 0) -mu."""
        out = []
        for mu in sorted({mu for (mu, _) in self.plans.keys}):
            out.append(mu)
            if mu > 0:
                out.append(self.N - mu)
        return out

    def legendre_synthesis_bins(self, beta: np.ndarray) -> np.ndarray:
        """beta (B, 4l^2) (only the plan set's orders are read) -> g (B, 2l, nbins)
        on range_bins(); same arithmetic as legendre_synthesis."""
        l = self.l
        beta = np.atleast_2d(beta)
        B = beta.shape[0]
        ins = [chain_rhs(l, beta, mu, p) for (mu, p) in self.plans.keys]
        outs, _ = self.plans.apply_all(ins, transpose=False, nthreads=self.nthreads)
        u = dict(zip(self.plans.keys, outs))
        bins = self.range_bins()
        col = {b: i for i, b in enumerate(bins)}
        g = np.zeros((B, 2 * l, len(bins)), dtype=np.complex128)
        isr = 1.0 / np.sqrt(self.rho)
        for mu in sorted({mu for (mu, _) in self.plans.keys}):
            ue = u[(mu, 0)]
            uo = u.get((mu, 1), np.zeros_like(ue))
            gp = (ue + uo) * isr[:, None]
            gm = (ue - uo) * isr[:, None]
            signs = (0,) if mu == 0 else (0, 1)
            c = 0
            for b in range(B):
                for s in signs:
                    j = col[mu if s == 0 else self.N - mu]
                    g[b, l:, j] = gp[:, c] + 1j * gp[:, c + 1]
                    g[b, :l, j] = (gm[:, c] + 1j * gm[:, c + 1])[::-1]
                    c += 2
        return g

    def legendre_analysis_bins(self, gbins: np.ndarray, beta_out: np.ndarray) -> None:
        """Unnormalised DFT values on range_bins() (B, 2l, nbins) -> the plan set's
        coefficients written into beta_out (B, 4l^2); same arithmetic as
        legendre_analysis."""
        l, N = self.l, self.N
        B = gbins.shape[0]
        col = {b: i for i, b in enumerate(self.range_bins())}
        hs = np.sqrt(self.rho) / 2.0
        ins = []
        for (mu, p) in self.plans.keys:
            signs = (0,) if mu == 0 else (0, 1)
            cols = []
            for b in range(B):
                for s in signs:
                    j = col[mu if s == 0 else N - mu]
                    gp = gbins[b, l:, j] / N
                    gm = gbins[b, :l, j][::-1] / N
                    uu = ((gp + gm) if p == 0 else (gp - gm)) * hs
                    cols.append(uu.real)
                    cols.append(uu.imag)
            ins.append(np.stack(cols, axis=1))
        outs, _ = self.plans.apply_all(ins, transpose=True, nthreads=self.nthreads)
        for (mu, p), o in zip(self.plans.keys, outs):
            scatter_rhs(l, beta_out, mu, p, o)

    # Full transforms -----------------------------------------------------------
    def synthesize(self, beta: np.ndarray) -> np.ndarray:
        g, _ = self.legendre_synthesis(beta)
        return np.fft.ifft(g, axis=-1) * self.N  # sum_m g_m e^{+2 pi i m n / N}

    def analyze(self, grid: np.ndarray) -> np.ndarray:
        beta, _ = self.legendre_analysis(np.fft.fft(np.asarray(grid), axis=-1))
        return beta


def random_coefficients(l: int, batch: int, seed: int, decaying_member: int | None = None) -> np.ndarray:
    """Seeded i.i.d. N(0,1) real and imaginary parts; optionally one
    member scaled by (k+1)^-2 (BASELINE.json config 3)."""
    rng = np.random.default_rng(seed)
    beta = rng.standard_normal((batch, 4 * l * l)) + 1j * rng.standard_normal((batch, 4 * l * l))
    if decaying_member is not None:
        k = np.empty(4 * l * l)
        for m in range(-(2 * l - 1), 2 * l):
            o = coeff_offset(l, m)
            mu = abs(m)
            k[o:o + 2 * l - mu] = np.arange(mu, 2 * l)
        beta[decaying_member] *= (k + 1.0) ** -2
    return beta


def dense_synthesis(l: int, beta: np.ndarray, cos_theta: np.ndarray) -> np.ndarray:
    """Independent O(l^3) synthesis with scipy (small l only): f(theta_t, phi_n)."""
    from scipy.special import lpmv, gammaln
    N = 4 * l - 1
    beta = np.atleast_2d(beta)
    x = np.asarray(cos_theta)
    phi = 2 * np.pi * np.arange(N) / N
    f = np.zeros((beta.shape[0], x.size, N), dtype=np.complex128)
    for m in range(-(2 * l - 1), 2 * l):
        mu = abs(m)
        for k in range(mu, 2 * l):
            # orthonormal on [-1, 1]: sqrt((2k+1)/2 (k-mu)!/(k+mu)!) P_k^mu, Condon-Shortley removed
            norm = np.sqrt((2 * k + 1) / 2.0 * np.exp(gammaln(k - mu + 1) - gammaln(k + mu + 1)))
            pb = norm * lpmv(mu, k, x) * (-1) ** mu
            c = beta[:, coeff_offset(l, m) + k - mu]
            f += c[:, None, None] * pb[None, :, None] * np.exp(1j * m * phi)[None, None, :]
    return f


def pbar_rows_extended(l, mu, x):
    """Pbar^mu_k(x) for k = mu .. 2l-1 (rows) at the points x, orthonormal on
    [-1, 1] without the Condon-Shortley phase (as oracle.sht_oracle.dense_synthesis),
    by the normalised three-term recurrence in extended precision."""
    x = np.asarray(x, dtype=np.longdouble)
    one = np.longdouble(1)
    p = np.full(x.shape, np.sqrt(np.longdouble(0.5)))
    for j in range(1, mu + 1):
        p = p * np.sqrt((2 * j + one) / (2 * j)) * np.sqrt(1 - x * x)
    out = [p]
    prev = np.zeros_like(p)
    for k in range(mu, 2 * l - 1):
        a = np.sqrt((4 * (k + one) ** 2 - 1) / ((k + one) ** 2 - mu * mu))
        b = np.sqrt((2 * k + 3) / (2 * k - one) * (k * k - mu * mu) / ((k + one) ** 2 - mu * mu)) if k > mu else 0
        nxt = a * x * out[-1] - b * prev
        prev = out[-1]
        out.append(nxt)
    return np.stack(out)
