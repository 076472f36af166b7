"""Butterfly plans and their GPU application — the reference's bfly:: API.

Mirrors the reference's public surface for the hot path
(/root/reference/proj/include/bfly/butterfly.hpp:86-100 and
include/bfly/transform.hpp:60-73):

=====================================  ============================================
reference                              here
=====================================  ============================================
bfly::build_plan(source, eps, C)       ``build_plan(dense, eps, C)``,
                                       ``build_glrow_plan(l, mu, parity, eps, C)``
bfly::apply(plan, v)                   ``apply(plan, v)``  (CUDA engine)
bfly::apply_transpose(plan, w)         ``apply_transpose(plan, w)``  (CUDA engine)
bfly::plan_stats(plan)                 ``plan_stats(plan)``
bfly::save_plan / load_plan            ``ButterflyPlan.to_bfly1`` / ``from_bfly1``
transform::forward / inverse           ``forward`` / ``inverse`` (aliases of apply)
=====================================  ============================================

Arguments keep the reference's meaning and errors: a wrong vector length
raises ``ValueError`` (the reference's ``std::invalid_argument``) with the
reference's message.  ``PlanSet`` is the batched form: many plans uploaded
once, applied to many right-hand sides in one launch.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, dptr, lib


@dataclass
class PlanStats:
    k_max: int
    k_avg: float
    k_sigma: float
    id_count: int
    levels: int
    stored_words: int
    m_max_words: int


class ButterflyPlan:
    """Host-side butterfly plan (the reference's ``bfly::ButterflyPlan``)."""

    def __init__(self, handle: int):
        if not handle:
            raise ValueError("null plan handle")
        self._h = C.c_void_p(handle)
        self._dev = None  # cached single-plan device set (uploaded once)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            self._dev = None
            lib().bfly_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # -- construction ------------------------------------------------------
    @classmethod
    def from_bfly1(cls, blob: bytes) -> "ButterflyPlan":
        """load_plan: parse the reference's BFLY1 bytes."""
        out = C.c_void_p()
        check(lib().bfly_plan_from_bfly1(blob, len(blob), C.byref(out)))
        return cls(out.value)

    def to_bfly1(self) -> bytes:
        """save_plan: the reference's BFLY1 bytes."""
        n = C.c_size_t(0)
        check(lib().bfly_plan_to_bfly1(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().bfly_plan_to_bfly1(self._h, buf, n.value, C.byref(n)))
        return buf.raw

    # -- introspection -----------------------------------------------------
    def info(self) -> dict:
        info = (C.c_int64 * 10)()
        ks = (C.c_double * 2)()
        check(lib().bfly_plan_info(self._h, info, ks))
        keys = ["n_rows", "n_cols", "levels", "stored_words", "m_max_words", "events",
                "root_groups", "k_max", "id_count", "block_width"]
        d = {k: int(v) for k, v in zip(keys, info)}
        d["k_avg"], d["k_sigma"] = float(ks[0]), float(ks[1])
        return d

    @property
    def n_rows(self) -> int:
        return self.info()["n_rows"]

    @property
    def n_cols(self) -> int:
        return self.info()["n_cols"]

    def device_set(self, device: int = 0) -> "PlanSet":
        if self._dev is None or self._dev.device != device:
            self._dev = PlanSet([self], device=device)
        return self._dev


def build_plan(a: np.ndarray, eps: float, block_width: int = 60) -> ButterflyPlan:
    """bfly::build_plan over a DenseColumnSource (column_source.hpp:21-40)."""
    a = np.asfortranarray(a, dtype=np.float64)
    out = C.c_void_p()
    check(lib().bfly_plan_build_dense(dptr(a), a.shape[0], a.shape[1], float(eps), int(block_width),
                                      C.byref(out)))
    return ButterflyPlan(out.value)


def build_glrow_plan(l: int, mu: int, parity: int, eps: float, block_width: int = 60) -> ButterflyPlan:
    """Plan of A(i, j) = sqrt(rho_i) Pbar^mu_{mu+2j+parity}(x_i) on the l positive GL nodes."""
    out = C.c_void_p()
    check(lib().bfly_plan_build_glrow(l, mu, parity, float(eps), int(block_width), C.byref(out)))
    return ButterflyPlan(out.value)


def build_glrow_planset(l: int, eps: float, block_width: int = 60, mu_range=None,
                        threads: int | None = None, rule=None) -> list[ButterflyPlan]:
    """Every non-empty (mu, parity) plan, mu in mu_range (default [0, 2l)), built on host threads.
    rule: optional (nodes, rho) of length l (default this library's GL rule)."""
    import os
    mu0, mu1 = mu_range if mu_range is not None else (0, 2 * l)
    threads = threads or os.cpu_count() or 1
    n = C.c_int(0)
    count = sum(1 for mu in range(mu0, mu1) for p in (0, 1) if chain_cols(l, mu, p) > 0)
    arr = (C.c_void_p * count)()
    if rule is None:
        check(lib().bfly_glrow_planset_build(l, mu0, mu1, float(eps), block_width, threads, arr, count,
                                             C.byref(n)))
    else:
        nodes = np.ascontiguousarray(rule[0], dtype=np.float64)
        rho = np.ascontiguousarray(rule[1], dtype=np.float64)
        if nodes.shape != (l,) or rho.shape != (l,):
            raise ValueError(f"rule: expected {l} nodes and weights")
        dp = C.POINTER(C.c_double)
        check(lib().bfly_glrow_planset_build_rule(l, mu0, mu1, float(eps), block_width, threads,
                                                  nodes.ctypes.data_as(dp), rho.ctypes.data_as(dp), arr, count,
                                                  C.byref(n)))
    assert n.value == count
    return [ButterflyPlan(arr[i]) for i in range(count)]


def chain_cols(l: int, mu: int, parity: int) -> int:
    """n_p(mu): columns of chain p at order mu (SURVEY.md §8 definitions)."""
    n = (2 * l - mu + 1) // 2 if parity == 0 else (2 * l - mu) // 2
    return max(n, 0)


def plan_stats(plan: ButterflyPlan) -> PlanStats:
    """bfly::plan_stats (reference src/butterfly.cpp:515-541)."""
    i = plan.info()
    return PlanStats(i["k_max"], i["k_avg"], i["k_sigma"], i["id_count"], i["levels"],
                     i["stored_words"], i["m_max_words"])


class PlanSet:
    """Plans compiled into one device program and uploaded once.

    ``apply(x, transpose)`` applies every plan to ``nrhs`` right-hand sides in
    one engine launch.  Layout (stacked, column-major per plan): plan p's block
    is (n_in(p), nrhs) starting at nrhs * sum_{q<p} n_in(q).
    """

    def __init__(self, plans: list[ButterflyPlan], device: int = 0):
        self.device = device
        self.plans = list(plans)  # keep host plans alive
        arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
        out = C.c_void_p()
        check(lib().bfly_dev_planset_create(arr, len(plans), device, C.byref(out)))
        self._h = out
        shapes = [p.info() for p in plans]
        self.rows = [s["n_rows"] for s in shapes]
        self.cols = [s["n_cols"] for s in shapes]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            lib().bfly_dev_planset_destroy(h)
            self._h = None

    def info(self) -> dict:
        info = (C.c_int64 * 8)()
        check(lib().bfly_dev_planset_info(self._h, info))
        keys = ["n_plans", "n_jobs", "stored_words", "fetched_bytes", "stream_bytes", "arena_cells",
                "smem_bytes", "total_rows"]
        return {k: int(v) for k, v in zip(keys, info)}

    def apply_device(self, x, out, nrhs: int, transpose: bool = False, stream=None) -> None:
        """Device pointers (torch CUDA tensors, float64, contiguous)."""
        st = stream if stream is not None else _current_stream(self.device)
        check(lib().bfly_dev_apply(self._h, int(transpose), C.c_void_p(x.data_ptr()), x.numel(),
                                   C.c_void_p(out.data_ptr()), out.numel(), int(nrhs), st))

    def apply_host(self, x: np.ndarray, nrhs: int, transpose: bool = False) -> np.ndarray:
        """Host numpy buffers (copied to and from the device inside)."""
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        n_out = (sum(self.cols) if transpose else sum(self.rows)) * nrhs
        out = np.empty(n_out)
        check(lib().bfly_host_apply(self._h, int(transpose), dptr(x), x.size, dptr(out), out.size,
                                    int(nrhs)))
        return out

    def stack(self, blocks: list[np.ndarray]) -> tuple[np.ndarray, int]:
        nrhs = blocks[0].shape[1]
        return np.concatenate([np.asfortranarray(b).ravel(order="F") for b in blocks]), nrhs

    def unstack(self, flat: np.ndarray, nrhs: int, transpose: bool) -> list[np.ndarray]:
        sizes = self.cols if transpose else self.rows
        out, at = [], 0
        for n in sizes:
            out.append(flat[at:at + n * nrhs].reshape((n, nrhs), order="F"))
            at += n * nrhs
        return out


def _current_stream(device: int):
    try:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    except ImportError:
        pass
    return None


def _apply(plan: ButterflyPlan, v, transpose: bool):
    info = plan.info()
    n_in = info["n_rows"] if transpose else info["n_cols"]
    who = "apply_transpose" if transpose else "apply"
    try:
        import torch
        is_torch = isinstance(v, torch.Tensor)
    except ImportError:
        is_torch = False
    if is_torch and v.is_cuda:
        vv = v.reshape(v.shape[0], -1) if v.dim() > 1 else v.reshape(-1, 1)
        if vv.shape[0] != n_in:
            raise _lib.BflyInvalidArgument(_lib.BFLY_EINVAL,
                                           f"{who}: vector length {vv.shape[0]}, expected {n_in}")
        nrhs = vv.shape[1]
        x = vv.t().contiguous().to(torch.float64)  # column-major (n_in x nrhs)
        n_out = info["n_cols"] if transpose else info["n_rows"]
        out = torch.empty(nrhs * n_out, dtype=torch.float64, device=v.device)
        plan.device_set(v.device.index or 0).apply_device(x, out, nrhs, transpose)
        res = out.view(nrhs, n_out).t()
        return res.reshape(-1) if v.dim() == 1 else res
    a = np.asarray(v, dtype=np.float64)
    vv = a.reshape(-1, 1) if a.ndim == 1 else a
    if vv.shape[0] != n_in:
        raise _lib.BflyInvalidArgument(_lib.BFLY_EINVAL,
                                       f"{who}: vector length {vv.shape[0]}, expected {n_in}")
    ps = plan.device_set(0)
    flat = ps.apply_host(np.asfortranarray(vv).ravel(order="F"), vv.shape[1], transpose)
    res = ps.unstack(flat, vv.shape[1], transpose)[0]
    return res[:, 0] if a.ndim == 1 else res


def apply(plan: ButterflyPlan, v):
    """bfly::apply — A v on the GPU (v: numpy 1-D/2-D or torch CUDA tensor)."""
    return _apply(plan, v, False)


def apply_transpose(plan: ButterflyPlan, w):
    """bfly::apply_transpose — A^T w on the GPU."""
    return _apply(plan, w, True)


# transform::forward / transform::inverse delegate to apply / apply_transpose
# (reference src/transform.cpp:83-91).
forward = apply
inverse = apply_transpose
