"""Spherical harmonic transforms on the GPU (bandlimit l, all orders m).

Synthesis ("inverse SHT" in arXiv 0910.5435 §2) maps coefficients beta_k^m to
values on the 2l x (4l-1) Gauss-Legendre x equispaced grid; analysis maps grid
values back.  Per order |m| = mu the Legendre stage is the reference's
transform::forward / transform::inverse (bfly::apply / apply_transpose,
/root/reference/proj/src/transform.cpp:83-91) on the GL-row plans of both
degree parities, executed for every mu in one launch (whole-chain engine for single
functions; for batches the wave program as one dependency-ordered persistent launch,
csrc/wgraph.cu); the phi stage is the fused in-SM
DFT of length 4l-1 (csrc/phi.cu; Rader's algorithm for prime lengths, cuFFT
only for the stage-wise entry points).

Layouts (complex128), see include/bfly_b200.h:
  coefficients: per function 4 l^2 values, order-major:
      m = 0 (k = 0..2l-1), then for mu = 1..2l-1: m = +mu (k = mu..2l-1),
      m = -mu (k = mu..2l-1)
  grid: per function (2l, 4l-1), rows ordered by increasing cos(theta).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import check, dptr, lib
from .butterfly import ButterflyPlan, _current_stream


def coeff_offset(l: int, m: int) -> int:
    """Index of beta_{|m|}^m in the packed per-function coefficient vector."""
    mu = abs(m)
    if mu > 2 * l - 1:
        raise ValueError(f"|m| = {mu} exceeds 2l-1 = {2 * l - 1}")
    base = 0 if mu == 0 else 2 * l + (mu - 1) * (4 * l - mu)
    return base + (2 * l - mu if m < 0 else 0)


def coeff_index(l: int, m: int, k: int) -> int:
    if not abs(m) <= k <= 2 * l - 1:
        raise ValueError(f"(k={k}, m={m}) outside the bandlimit l={l}")
    return coeff_offset(l, m) + (k - abs(m))


def half_offset(l: int, m: int) -> int:
    """Real fields: first coefficient of order m >= 0 in the half layout."""
    if not 0 <= m < 2 * l:
        raise ValueError(f"order {m} outside [0, {2 * l})")
    return m * 2 * l - m * (m - 1) // 2


def half_from_full(l: int, beta: np.ndarray) -> np.ndarray:
    """The m >= 0 blocks of packed coefficients (..., 4l^2) -> (..., l(2l+1))."""
    out = np.empty(beta.shape[:-1] + (l * (2 * l + 1),), dtype=np.complex128)
    for m in range(2 * l):
        o, h = coeff_offset(l, m), half_offset(l, m)
        out[..., h:h + 2 * l - m] = beta[..., o:o + 2 * l - m]
    return out


def full_from_half(l: int, half: np.ndarray) -> np.ndarray:
    """Real-field coefficients: beta^{-m} = conj(beta^m), Im beta^0 = 0."""
    out = np.empty(half.shape[:-1] + (4 * l * l,), dtype=np.complex128)
    for m in range(2 * l):
        h = half_offset(l, m)
        blk = half[..., h:h + 2 * l - m]
        if m == 0:
            blk = blk.real.astype(np.complex128)
        out[..., coeff_offset(l, m):coeff_offset(l, m) + 2 * l - m] = blk
        if m > 0:
            out[..., coeff_offset(l, -m):coeff_offset(l, -m) + 2 * l - m] = np.conj(blk)
    return out


def pack_dense(l: int, dense: np.ndarray) -> np.ndarray:
    """(..., 2l, 4l-1) array indexed [k, m + 2l - 1] -> packed (..., 4l^2)."""
    lead = dense.shape[:-2]
    out = np.zeros(lead + (4 * l * l,), dtype=np.complex128)
    for m in range(-(2 * l - 1), 2 * l):
        mu = abs(m)
        o = coeff_offset(l, m)
        out[..., o:o + 2 * l - mu] = dense[..., mu:2 * l, m + 2 * l - 1]
    return out


def unpack_dense(l: int, packed: np.ndarray) -> np.ndarray:
    lead = packed.shape[:-1]
    out = np.zeros(lead + (2 * l, 4 * l - 1), dtype=np.complex128)
    for m in range(-(2 * l - 1), 2 * l):
        mu = abs(m)
        o = coeff_offset(l, m)
        out[..., mu:2 * l, m + 2 * l - 1] = packed[..., o:o + 2 * l - mu]
    return out


def _rule_arrays(l: int, rule):
    if rule is None:
        return None, None
    nodes = np.ascontiguousarray(rule[0], dtype=np.float64)
    rho = np.ascontiguousarray(rule[1], dtype=np.float64)
    if nodes.shape != (l,) or rho.shape != (l,):
        raise ValueError(f"rule: expected {l} nodes and weights")
    return nodes, rho


class SHT:
    """GPU spherical harmonic transform of bandlimit l (plans uploaded once)."""

    def __init__(self, l: int, eps: float = 1e-12, block_width: int = 60, threads: int | None = None,
                 device: int = 0, _handle=None, rule=None):
        """rule: optional (nodes, rho) quadrature of length l (e.g. the
        reference's build_rule(0, l, even)); default this library's GL rule."""
        self.l = l
        self.N = 4 * l - 1
        self.device = device
        if _handle is None:
            out = C.c_void_p()
            threads = threads or os.cpu_count() or 1
            nodes, rho = _rule_arrays(l, rule)
            check(lib().bfly_sht_create_rule(l, float(eps), int(block_width), int(threads),
                                             dptr(nodes) if nodes is not None else None,
                                             dptr(rho) if rho is not None else None, device, C.byref(out)))
            _handle = out
        self._h = _handle

    @classmethod
    def from_plans(cls, l: int, plans: list[ButterflyPlan], rho: np.ndarray | None = None,
                   device: int = 0) -> "SHT":
        """Use caller-built plans (e.g. the reference's, via BFLY1) in (mu, parity) order."""
        arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
        out = C.c_void_p()
        rp = None
        if rho is not None:
            rho = np.ascontiguousarray(rho, dtype=np.float64)
            rp = dptr(rho)
        check(lib().bfly_sht_create_from_plans(l, arr, len(plans), rp, device, C.byref(out)))
        obj = cls(l, device=device, _handle=out)
        obj._plans = plans
        return obj

    @classmethod
    def range(cls, l: int, mu_begin: int, mu_end: int, eps: float = 1e-12, block_width: int = 60,
              threads: int | None = None, device: int = 0, plans: list[ButterflyPlan] | None = None,
              rule=None, rho: np.ndarray | None = None) -> "SHT":
        """Legendre stage of the orders [mu_begin, mu_end) only (one shard of the
        order-sharded transform, paper_0910_5435_b200/sharded.py).  Coefficients
        keep the packed 4l^2 layout and the bins the (4l-1, B, 2l) layout; only
        the range's entries are read or written.  The phi stage needs all
        orders, so the full-transform entry points reject a partial range."""
        from .butterfly import build_glrow_planset
        if plans is None:
            plans = build_glrow_planset(l, eps, block_width, mu_range=(mu_begin, mu_end), threads=threads,
                                        rule=rule)
        if rho is None and rule is not None:
            rho = rule[1]
        if rho is not None:
            rho = np.ascontiguousarray(rho, dtype=np.float64)
        arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
        out = C.c_void_p()
        check(lib().bfly_sht_create_range(l, mu_begin, mu_end, arr, len(plans),
                                          dptr(rho) if rho is not None else None, device, C.byref(out)))
        obj = cls(l, device=device, _handle=out)
        obj._plans = plans
        obj.mu_range = (mu_begin, mu_end)
        return obj

    def save(self, path: str) -> None:
        """Write the device-ready packed program (reload with SHT.load, no plan build)."""
        check(lib().bfly_sht_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str, device: int = 0) -> "SHT":
        out = C.c_void_p()
        check(lib().bfly_sht_load(os.fsencode(path), device, C.byref(out)))
        info = (C.c_int64 * 8)()
        check(lib().bfly_sht_info(out, info))
        return cls(int(info[0]), device=device, _handle=out)

    def __del__(self):
        h = getattr(self, "_h", None)
        if getattr(self, "_borrowed", False):  # owned by another handle (e.g. a shard)
            return
        if h is not None and h.value and _lib._lib is not None:
            lib().bfly_sht_destroy(h)
            self._h = None

    # -- metadata ----------------------------------------------------------
    def info(self) -> dict:
        info = (C.c_int64 * 8)()
        check(lib().bfly_sht_info(self._h, info))
        keys = ["l", "n_plans", "stored_words", "fetched_bytes", "n_jobs", "smem_bytes", "coeffs",
                "grid_points"]
        return {k: int(v) for k, v in zip(keys, info)}

    def program_info(self) -> dict:
        """Programs held by the handle (whole-chain engine and/or wave programs)
        and the wave layout (bfly_sht_program_info)."""
        info = (C.c_int64 * 10)()
        check(lib().bfly_sht_program_info(self._h, info))
        keys = ["whole", "waves", "levels", "root_groups", "v_cells", "nodes", "event_words", "wave_min_batch",
                "graph", "graph_groups"]
        return {k: int(v) for k, v in zip(keys, info)}

    def uses_waves(self, batch: int) -> bool:
        """Whether a call with `batch` functions runs on the wave programs."""
        p = self.program_info()
        return bool(p["waves"]) and (not p["whole"] or batch >= p["wave_min_batch"])

    def engine_time(self, enable: bool) -> tuple[list[float], list[int]]:
        """Summed CUDA-event time (ms) and count of the engine launches since the
        last call, per direction (synthesis, analysis); then switch timing on/off."""
        ms = (C.c_double * 2)()
        n = (C.c_int64 * 2)()
        check(lib().bfly_sht_engine_time(self._h, int(enable), ms, n))
        return [ms[0], ms[1]], [int(n[0]), int(n[1])]

    def rule(self) -> tuple[np.ndarray, np.ndarray]:
        nodes = np.empty(self.l)
        rho = np.empty(self.l)
        check(lib().bfly_sht_rule(self._h, dptr(nodes), dptr(rho)))
        return nodes, rho

    def cos_theta(self) -> np.ndarray:
        """cos(theta_t), t = 0..2l-1, increasing (grid row order)."""
        nodes, _ = self.rule()
        return np.concatenate([-nodes[::-1], nodes])

    @property
    def n_coeffs(self) -> int:
        return 4 * self.l * self.l

    @property
    def grid_shape(self) -> tuple[int, int]:
        return (2 * self.l, self.N)

    # -- device API (torch CUDA tensors, complex128) -------------------------
    def _check(self, t, tail, name):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.complex128):
            raise TypeError(f"{name}: expected a CUDA complex128 tensor")
        if t.device.index != self.device:
            raise ValueError(f"{name}: tensor on {t.device}, the handle is on cuda:{self.device}")
        if tuple(t.shape[-len(tail):]) != tuple(tail):
            raise ValueError(f"{name}: trailing shape {tuple(t.shape)}, expected (..., {tail})")
        if not t.is_contiguous():
            raise ValueError(f"{name}: tensor must be contiguous")

    def _check_out(self, out, shape, name, dtype=None):
        """A caller-supplied output must be exactly what the kernels write:
        contiguous, on this handle's device, of the right dtype and shape (the
        CUDA side trusts the pointer, so anything smaller would be overrun)."""
        import torch
        dtype = dtype or torch.complex128
        if not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == dtype):
            raise TypeError(f"{name}: out must be a CUDA {dtype} tensor")
        if out.device.index != self.device:
            raise ValueError(f"{name}: out on {out.device}, the handle is on cuda:{self.device}")
        if tuple(out.shape) != tuple(shape):
            raise ValueError(f"{name}: out has shape {tuple(out.shape)}, expected {tuple(shape)}")
        if not out.is_contiguous():
            raise ValueError(f"{name}: out must be contiguous")

    def synthesize(self, beta, out=None, stream=None):
        """beta (B, 4l^2) -> grid (B, 2l, 4l-1)."""
        import torch
        self._check(beta, (self.n_coeffs,), "synthesize")
        B = beta.numel() // self.n_coeffs
        if out is None:
            out = torch.empty(beta.shape[:-1] + self.grid_shape, dtype=torch.complex128, device=beta.device)
        self._check_out(out, beta.shape[:-1] + self.grid_shape, "synthesize")
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_synthesize(self._h, C.c_void_p(beta.data_ptr()), C.c_void_p(out.data_ptr()),
                                        B, st))
        return out

    def analyze(self, grid, out=None, stream=None):
        """grid (B, 2l, 4l-1) -> beta (B, 4l^2)."""
        import torch
        self._check(grid, self.grid_shape, "analyze")
        B = grid.numel() // (2 * self.l * self.N)
        if out is None:
            out = torch.empty(grid.shape[:-2] + (self.n_coeffs,), dtype=torch.complex128, device=grid.device)
        self._check_out(out, grid.shape[:-2] + (self.n_coeffs,), "analyze")
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_analyze(self._h, C.c_void_p(grid.data_ptr()), C.c_void_p(out.data_ptr()),
                                     B, st))
        return out

    # -- real fields (beta^{-m} = conj(beta^m), Im beta^0 = 0) -----------------
    @property
    def n_coeffs_half(self) -> int:
        return self.l * (2 * self.l + 1)

    def synthesize_real(self, beta_half, out=None, stream=None):
        """Half-layout coefficients (B, l(2l+1)) complex128 -> real grid (B, 2l, 4l-1) float64."""
        import torch
        self._check(beta_half, (self.n_coeffs_half,), "synthesize_real")
        B = beta_half.numel() // self.n_coeffs_half
        if out is None:
            out = torch.empty(beta_half.shape[:-1] + self.grid_shape, dtype=torch.float64, device=beta_half.device)
        self._check_out(out, beta_half.shape[:-1] + self.grid_shape, "synthesize_real", torch.float64)
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_synthesize_real(self._h, C.c_void_p(beta_half.data_ptr()), C.c_void_p(out.data_ptr()),
                                             B, st))
        return out

    def analyze_real(self, grid, out=None, stream=None):
        """Real grid (B, 2l, 4l-1) float64 -> half-layout coefficients (B, l(2l+1))."""
        import torch
        if not (isinstance(grid, torch.Tensor) and grid.is_cuda and grid.dtype == torch.float64
                and grid.is_contiguous() and tuple(grid.shape[-2:]) == self.grid_shape
                and grid.device.index == self.device):
            raise ValueError("analyze_real: expected a contiguous CUDA float64 (..., 2l, 4l-1) tensor "
                             f"on cuda:{self.device}")
        B = grid.numel() // (2 * self.l * self.N)
        if out is None:
            out = torch.empty(grid.shape[:-2] + (self.n_coeffs_half,), dtype=torch.complex128, device=grid.device)
        self._check_out(out, grid.shape[:-2] + (self.n_coeffs_half,), "analyze_real")
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_analyze_real(self._h, C.c_void_p(grid.data_ptr()), C.c_void_p(out.data_ptr()), B, st))
        return out

    def phi_shape(self, batch: int) -> tuple[int, int, int]:
        """Shape of the phi-stage buffer: (4l-1 bins, batch, 2l latitude rows)."""
        return (self.N, batch, 2 * self.l)

    def _check_phi(self, t, name):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.complex128 and t.dim() == 3
                and t.shape[0] == self.N and t.shape[2] == 2 * self.l and t.is_contiguous()
                and t.device.index == self.device):
            raise ValueError(f"{name}: expected a contiguous CUDA complex128 tensor of shape "
                             f"({self.N}, batch, {2 * self.l})")
        return t.shape[1]

    def legendre_synthesize(self, beta, out=None, stream=None):
        """Legendre stage only: beta (B, 4l^2) -> g_m(theta_t) as (4l-1, B, 2l) [bin][b][t]."""
        import torch
        self._check(beta, (self.n_coeffs,), "legendre_synthesize")
        B = beta.numel() // self.n_coeffs
        if out is None:
            out = torch.empty(self.phi_shape(B), dtype=torch.complex128, device=beta.device)
        self._check_out(out, self.phi_shape(B), "legendre_synthesize")
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_legendre_synthesize(self._h, C.c_void_p(beta.data_ptr()),
                                                 C.c_void_p(out.data_ptr()), B, st))
        return out

    def legendre_analyze(self, gdft, out=None, stream=None):
        """Legendre stage only: unnormalised forward DFT (4l-1, B, 2l) -> beta (B, 4l^2)."""
        import torch
        B = self._check_phi(gdft, "legendre_analyze")
        if out is None:
            out = torch.empty((B, self.n_coeffs), dtype=torch.complex128, device=gdft.device)
        self._check_out(out, (B, self.n_coeffs), "legendre_analyze")
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_legendre_analyze(self._h, C.c_void_p(gdft.data_ptr()),
                                              C.c_void_p(out.data_ptr()), B, st))
        return out

    def phi_synthesize(self, gbins, out=None, stream=None):
        """phi stage only: (4l-1, B, 2l) bins -> grid (B, 2l, 4l-1)."""
        import torch
        B = self._check_phi(gbins, "phi_synthesize")
        if out is None:
            out = torch.empty((B,) + self.grid_shape, dtype=torch.complex128, device=gbins.device)
        self._check_out(out, (B,) + self.grid_shape, "phi_synthesize")
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_phi_synthesize(self._h, C.c_void_p(gbins.data_ptr()), C.c_void_p(out.data_ptr()),
                                            B, st))
        return out

    def phi_analyze(self, grid, out=None, stream=None):
        """phi stage only: grid (B, 2l, 4l-1) -> unnormalised forward DFT (4l-1, B, 2l)."""
        import torch
        self._check(grid, self.grid_shape, "phi_analyze")
        B = grid.numel() // (2 * self.l * self.N)
        if out is None:
            out = torch.empty(self.phi_shape(B), dtype=torch.complex128, device=grid.device)
        self._check_out(out, self.phi_shape(B), "phi_analyze")
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_sht_phi_analyze(self._h, C.c_void_p(grid.data_ptr()), C.c_void_p(out.data_ptr()),
                                         B, st))
        return out

    def synthesize_host_ptr(self, beta_ptr: int, grid_ptr: int, batch: int) -> None:
        """Host-buffer synthesis on raw (e.g. pinned) host pointers."""
        check(lib().bfly_sht_synthesize_host(self._h, C.cast(beta_ptr, C.POINTER(C.c_double)),
                                             C.cast(grid_ptr, C.POINTER(C.c_double)), batch))

    def analyze_host_ptr(self, grid_ptr: int, beta_ptr: int, batch: int) -> None:
        check(lib().bfly_sht_analyze_host(self._h, C.cast(grid_ptr, C.POINTER(C.c_double)),
                                          C.cast(beta_ptr, C.POINTER(C.c_double)), batch))

    # -- host API (numpy; copies inside, synchronous) -------------------------
    def synthesize_host(self, beta: np.ndarray) -> np.ndarray:
        beta = np.ascontiguousarray(beta, dtype=np.complex128)
        if beta.shape[-1] != self.n_coeffs:
            raise ValueError(f"synthesize: trailing size {beta.shape[-1]}, expected {self.n_coeffs}")
        B = beta.size // self.n_coeffs
        out = np.empty(beta.shape[:-1] + self.grid_shape, dtype=np.complex128)
        check(lib().bfly_sht_synthesize_host(self._h, dptr(beta.view(np.float64)),
                                             dptr(out.view(np.float64)), B))
        return out

    def analyze_host(self, grid: np.ndarray) -> np.ndarray:
        grid = np.ascontiguousarray(grid, dtype=np.complex128)
        if tuple(grid.shape[-2:]) != self.grid_shape:
            raise ValueError(f"analyze: trailing shape {grid.shape[-2:]}, expected {self.grid_shape}")
        B = grid.size // (2 * self.l * self.N)
        out = np.empty(grid.shape[:-2] + (self.n_coeffs,), dtype=np.complex128)
        check(lib().bfly_sht_analyze_host(self._h, dptr(grid.view(np.float64)),
                                          dptr(out.view(np.float64)), B))
        return out
