"""CPU interpreter of the wave programs — TEST INFRASTRUCTURE ONLY.

It replays the level-synchronous program that build_waves compiles
(paper_0910_5435_b200/csrc/waves.hpp; fetched through bfly_waves_inspect) with
the semantics of the tensor-core kernels (wavekern.cu, rootmma.cu), in numpy:
forward nodes level by level (c = z[sel] + T z[others]), root stripes
(rows += S c); transpose roots (c = S^T rows), then node pairs level by level
backwards (z[others] (=|+=) T^T c, z[sel] (=|+=) c, first node of a pair
assigns).  V starts as NaN, so a read of a cell no level wrote shows up in the
result.  This validates the host compiler (cell assignment, levels, aliasing of
full-rank leaves, copy nodes, pairs) on a machine without a GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_0910_5435_b200._lib import check, lib


def untile(data, off, rows, cols, nib):
    """A rows x cols matrix stored as 16 x 16 swizzled tiles (csrc/packer.hpp
    tiled_index: tile (ib, qb) at (qb nib + ib) 256, element (i, q) of a tile at
    q 16 + (i ^ 4 (q & 3)))."""
    i = np.arange(rows)[:, None]
    q = np.arange(cols)[None, :]
    pos = ((q >> 4) * nib + (i >> 4)) * 256 + (q & 15) * 16 + ((i & 15) ^ (4 * (q & 3)))
    return data[off + pos] if rows and cols else np.zeros((rows, cols), dtype=data.dtype)


class WaveProgram:
    def __init__(self, plans):
        arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
        sizes = (C.c_int64 * 10)()
        check(lib().bfly_waves_inspect(arr, len(plans), sizes, *([None] * 10)))
        nT, nidx, nnodes, nfwd, npairs, levels, vcells, nstripes, nS, aliased = [int(x) for x in sizes]
        self.T = np.zeros(max(nT, 1))
        self.idx = np.zeros(max(nidx, 1), np.uint32)
        nodes = np.zeros((max(nnodes, 1), 8), np.uint32)
        self.fwd = np.zeros(max(nfwd, 1), np.uint32)
        pairs = np.zeros((max(npairs, 1), 2), np.uint32)
        self.fwd_begin = np.zeros(levels + 1, np.uint32)
        self.bwd_begin = np.zeros(levels + 1, np.uint32)
        self.plan_in = np.zeros(len(plans), np.uint32)
        stripes = np.zeros((max(nstripes, 1), 8), np.uint64)
        self.S = np.zeros(max(nS, 1))
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        check(lib().bfly_waves_inspect(arr, len(plans), sizes, ptr(self.T), ptr(self.idx), ptr(nodes), ptr(self.fwd),
                                       ptr(pairs), ptr(self.fwd_begin), ptr(self.bwd_begin), ptr(self.plan_in),
                                       ptr(stripes), ptr(self.S)))
        self.nodes = [dict(t_off=int(n[0]) | (int(n[1]) << 32), rank=int(n[2]), nothers=int(n[3]), idx=int(n[4]),
                           cA=int(n[5]), level=int(n[6]), nib=int(n[7])) for n in nodes[:nnodes]]
        self.fwd = self.fwd[:nfwd]
        self.pairs = pairs[:npairs]
        self.stripes = [dict(s_off=int(s[0]), rows=int(s[1]), rank=int(s[2]), lds=int(s[3]), coff=int(s[4]),
                             plan=int(s[5]), group=int(s[6]), row0=int(s[7])) for s in stripes[:nstripes]]
        self.levels, self.v_cells, self.aliased = levels, vcells, aliased
        self.plans = plans

    def _node(self, n):
        T = untile(self.T, n["t_off"], n["rank"], n["nothers"], n["nib"])
        sel = self.idx[n["idx"]:n["idx"] + n["rank"]]
        oth = self.idx[n["idx"] + n["rank"]:n["idx"] + n["rank"] + n["nothers"]]
        return T, sel, oth

    def _S(self, s):
        return untile(self.S, s["s_off"], s["rows"], s["rank"], s["lds"])

    def apply(self, ins):
        """ins[p]: (n_cols(p), R) -> outs[p]: (n_rows(p), R)."""
        R = ins[0].shape[1]
        V = np.full((self.v_cells, R), np.nan)
        for p, x in enumerate(ins):
            V[self.plan_in[p]:self.plan_in[p] + x.shape[0]] = x
        for L in range(1, self.levels + 1):
            for i in self.fwd[self.fwd_begin[L - 1]:self.fwd_begin[L]]:
                n = self.nodes[i]
                assert n["level"] == L
                T, sel, oth = self._node(n)
                V[n["cA"]:n["cA"] + n["rank"]] = V[sel] + (T @ V[oth] if n["nothers"] else 0.0)
        outs = [np.zeros((pl.n_rows, R)) for pl in self.plans]
        for s in self.stripes:
            c = V[s["coff"]:s["coff"] + s["rank"]]
            rb = s["row0"] - sum(pl.n_rows for pl in self.plans[:s["plan"]])
            outs[s["plan"]][rb:rb + s["rows"]] += self._S(s) @ c
        return outs

    def apply_transpose(self, ins):
        """ins[p]: (n_rows(p), R) -> outs[p]: (n_cols(p), R)."""
        R = ins[0].shape[1]
        V = np.full((self.v_cells, R), np.nan)
        for s in self.stripes:
            rb = s["row0"] - sum(pl.n_rows for pl in self.plans[:s["plan"]])
            V[s["coff"]:s["coff"] + s["rank"]] = self._S(s).T @ ins[s["plan"]][rb:rb + s["rows"]]
        for L in range(self.levels, 0, -1):
            for a, b in self.pairs[self.bwd_begin[L - 1]:self.bwd_begin[L]]:
                for k, ni in enumerate((a, b)):
                    if ni == 0xFFFFFFFF:
                        break
                    n = self.nodes[ni]
                    T, sel, oth = self._node(n)
                    c = V[n["cA"]:n["cA"] + n["rank"]]
                    zo = T.T @ c if n["rank"] else np.zeros((n["nothers"], R))
                    if k == 0:
                        V[oth] = zo
                        V[sel] = c
                    else:
                        V[oth] += zo
                        V[sel] += c
        return [V[self.plan_in[p]:self.plan_in[p] + pl.n_cols].copy() for p, pl in enumerate(self.plans)]
