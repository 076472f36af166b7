"""CPU interpreter of the engine's device program — TEST INFRASTRUCTURE ONLY.

It replays the stage stream that pack_program produces (format:
paper_0910_5435_b200/csrc/engine_format.hpp) with the kernel's record
semantics, in numpy, bounds-checking every cell index and payload offset and
poisoning the arena with NaN so a read of a never-written cell shows up in the
result.  This validates the packer (arena lifetimes, assign/accumulate flags,
record order in both directions) on a machine without a GPU; the CUDA engine
itself is validated against the reference on the GPU (tests/*_gpu.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_0910_5435_b200._lib import check, lib

OP_LOADZ, OP_SEL, OP_TPANEL, OP_SPANEL, OP_CXCH = range(5)
F_ASSIGN_FWD, F_ASSIGN_BWD, F_SYNC_FWD, F_SYNC_BWD, F_BEGIN, F_END, F_ASSIGN_SEL_BWD, F_CLOAD_FWD = (
    1, 2, 4, 8, 16, 32, 64, 128)
REC = np.dtype([("op", "u1"), ("flags", "u1"), ("nr", "<u2"), ("nc", "<u2"), ("moff", "<u2"),
                ("data", "<u4"), ("zA", "<u4"), ("zB", "<u4"), ("kl", "<u4"), ("cA", "<u4"),
                ("ld", "<u2"), ("pslot", "<u2")])
JOB = np.dtype([("stage0", "<u8"), ("n_stages", "<u4"), ("n_plans", "<u2"), ("mu", "<u2"),
                ("plan", "<u4", 2), ("yA", "<u4", 2), ("n_rows", "<u4"), ("n_cols", "<u4", 2),
                ("parity", "<u4"), ("yin", "<u4"), ("yout", "<u4"), ("kind", "<u4"), ("pad", "<u4")])
assert REC.itemsize == 32 and JOB.itemsize == 64


class Program:
    def __init__(self, plans, split=None, parity=None):
        """split None: one job per plan (generic); 0 / 1: event / root program of the SHT split."""
        arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
        sizes = (C.c_int64 * 8)()
        par = (C.c_int * len(plans))(*(parity if parity is not None else [0] * len(plans)))
        self.plan_yoff = np.zeros(len(plans), np.uint32)
        self.plan_groups = np.zeros(len(plans), np.uint32)

        def call(*bufs):
            if split is None:
                check(lib().bfly_pack_inspect(arr, len(plans), *bufs, sizes))
            else:
                check(lib().bfly_pack_inspect_split(arr, len(plans), par, split, *bufs, sizes,
                                                    self.plan_yoff.ctypes.data_as(C.c_void_p),
                                                    self.plan_groups.ctypes.data_as(C.c_void_p)))

        call(None, None, None, None)
        nbytes, nst, njobs, self.arena_cells, self.zo_cells, self.smem_bytes = [int(v) for v in sizes[:6]]
        self.c_cells, self.y_rows = int(sizes[6]), int(sizes[7])
        self.stream = np.zeros(nbytes, np.uint8)
        self.stage_off = np.zeros(nst, np.uint64)
        self.stage_bytes = np.zeros(nst, np.uint32)
        self.jobs = np.zeros(njobs, JOB)
        call(self.stream.ctypes.data_as(C.c_void_p), self.stage_off.ctypes.data_as(C.c_void_p),
             self.stage_bytes.ctypes.data_as(C.c_void_p), self.jobs.ctypes.data_as(C.c_void_p))

    def stage(self, s):
        off = int(self.stage_off[s])
        nbytes = int(self.stage_bytes[s])
        raw = self.stream[off:off + nbytes]
        n_rec, used = np.frombuffer(raw[:8].tobytes(), "<u4")
        assert used == nbytes and nbytes % 16 == 0 and nbytes <= 65536, (s, used, nbytes)
        recs = np.frombuffer(raw[16:16 + 32 * int(n_rec)].tobytes(), REC)
        return raw, recs


class Emu:
    """Replays one job for RC right-hand sides; inputs / outputs per plan slot."""

    def __init__(self, prog: Program, job, RC: int, cbuf=None):
        self.p, self.j, self.RC = prog, job, RC
        self.arena = np.full((prog.arena_cells, RC), np.nan)
        self.cbuf = cbuf

    def cells(self, a, n):
        assert 0 <= a and a + n <= self.p.arena_cells, ("cell range", a, n, self.p.arena_cells)
        return slice(a, a + n)

    def zc(self, r, k):
        k = np.asarray(k, dtype=np.int64)
        c = np.where(k < r["kl"], r["zA"] + k, r["zB"] + k - r["kl"])
        assert np.all(c < self.p.arena_cells), "z cell out of range"
        return c

    @staticmethod
    def u16(raw, at, n):
        assert at + 2 * n <= raw.size, "payload overrun"
        return np.frombuffer(raw[at:at + 2 * n].tobytes(), "<u2").astype(np.int64)

    @staticmethod
    def f64(raw, at, n):
        assert at % 8 == 0 and at + 8 * n <= raw.size, "panel overrun"
        return np.frombuffer(raw[at:at + 8 * n].tobytes(), "<f8")

    def run(self, inputs, bwd: bool, want_y: bool = True):
        """inputs[slot]: (n_in, RC).  Returns outputs[slot]: (n_out, RC)."""
        j = self.j
        n_plans = int(j["n_plans"])
        outs = [np.full((int(j["n_cols"][s]) if bwd else int(j["n_rows"]), self.RC), np.nan)
                for s in range(n_plans)]
        if bwd and inputs[0] is not None:
            for s in range(n_plans):
                self.arena[self.cells(int(j["yA"][s]), int(j["n_rows"]))] = inputs[s]
        stages = range(int(j["stage0"]), int(j["stage0"]) + int(j["n_stages"]))
        acc = None
        zo = None
        for st in (reversed(stages) if bwd else stages):
            raw, recs = self.p.stage(st)
            for r in (recs[::-1] if bwd else recs):
                op, fl = int(r["op"]), int(r["flags"])
                nr, nc, data = int(r["nr"]), int(r["nc"]), int(r["data"])
                if op == OP_CXCH:
                    sl = self.cells(int(r["zA"]), nr)
                    off = int(r["zB"])
                    assert off + nr <= self.cbuf.shape[0], "C range"
                    load = bool(fl & F_CLOAD_FWD) != bwd
                    if load:
                        self.arena[sl] = self.cbuf[off:off + nr]
                    else:
                        self.cbuf[off:off + nr] = self.arena[sl]
                    continue
                if op == OP_LOADZ:
                    sl = self.cells(int(r["zA"]), nr)
                    rows = slice(int(r["zB"]), int(r["zB"]) + nr)
                    if not bwd:
                        self.arena[sl] = inputs[int(r["pslot"])][rows]
                    else:
                        outs[int(r["pslot"])][rows] = self.arena[sl]
                elif op == OP_SEL:
                    sel = self.u16(raw, data, nr)
                    zc = self.zc(r, sel)
                    c = self.cells(int(r["cA"]), nr)
                    if not bwd:
                        self.arena[c] = self.arena[zc]
                    elif fl & F_ASSIGN_BWD:
                        self.arena[zc] = self.arena[c]
                    else:
                        self.arena[zc] += self.arena[c]
                else:
                    tp = op == OP_TPANEL
                    ld = int(r["ld"])
                    assert ld >= nr and ld % 2 == 1, "leading dimension"
                    P = self.f64(raw, data + int(r["moff"]), ld * nc).reshape((nc, ld)).T[:nr]
                    oth = self.u16(raw, data, nc) if tp else None
                    sel_at = data + ((2 * nc + 7) & ~7)
                    if not bwd:
                        if fl & F_BEGIN:
                            if tp:
                                sel = self.u16(raw, sel_at, nr)
                                acc = self.arena[self.zc(r, sel)].copy()
                            else:
                                acc = np.zeros((nr, self.RC))
                        if tp:
                            acc = acc + P @ self.arena[self.zc(r, oth)]
                        else:
                            acc = acc + P @ self.arena[self.cells(int(r["cA"]), nc)]
                        if fl & F_END:
                            if tp:
                                self.arena[self.cells(int(r["cA"]), nr)] = acc
                            else:
                                y = self.cells(int(r["zA"]), nr)
                                self.arena[y] = acc if fl & F_ASSIGN_FWD else self.arena[y] + acc
                    else:
                        vin = self.arena[self.cells(int(r["cA"] if tp else r["zA"]), nr)]
                        o = P.T @ vin
                        tgt = self.zc(r, oth) if tp else np.arange(int(r["cA"]), int(r["cA"]) + nc)
                        assert np.all(tgt < self.p.arena_cells)
                        if fl & F_ASSIGN_BWD:
                            self.arena[tgt] = o
                        else:
                            self.arena[tgt] += o
                        if tp and fl & F_BEGIN:
                            sel = self.u16(raw, sel_at, nr)
                            zc = self.zc(r, sel)
                            if fl & F_ASSIGN_SEL_BWD:
                                self.arena[zc] = vin
                            else:
                                self.arena[zc] += vin
        if not bwd and want_y:
            for s in range(n_plans):
                outs[s] = self.arena[self.cells(int(j["yA"][s]), int(j["n_rows"]))].copy()
        return outs


def emulate_split(plans, parity, inputs, bwd: bool, RC: int = 4):
    """SHT-style split programs on the CPU: events + roots through the C buffer."""
    ev = Program(plans, split=0, parity=parity)
    ro = Program(plans, split=1, parity=parity)
    cbuf = np.full((max(ev.c_cells, 1), RC), np.nan)
    out = [None] * len(plans)
    if not bwd:
        for job in ev.jobs:
            e = Emu(ev, job, RC, cbuf)
            e.run([inputs[int(job["plan"][0])]], False, want_y=False)
        ypart = np.full((max(ro.y_rows, 1), RC), np.nan)
        for job in ro.jobs:
            e = Emu(ro, job, RC, cbuf)
            y = e.run([None], False)[0]
            yo = int(job["yout"])
            ypart[yo:yo + y.shape[0]] = y
        for i, p in enumerate(plans):
            nr = p.n_rows
            yo, G = int(ro.plan_yoff[i]), int(ro.plan_groups[i])
            out[i] = sum(ypart[yo + g * nr: yo + (g + 1) * nr] for g in range(G))
    else:
        for job in ro.jobs:
            pi = int(job["plan"][0])
            yin, nr = int(job["yin"]), int(job["n_rows"])
            Emu(ro, job, RC, cbuf).run([inputs[pi][yin:yin + nr]], True)
        for job in ev.jobs:
            pi = int(job["plan"][0])
            out[pi] = Emu(ev, job, RC, cbuf).run([None], True)[0]
    return out, (ev, ro)


def emulate(plans, inputs, bwd: bool, RC: int = 4):
    """Apply every plan (one job per plan) on the CPU interpreter; inputs[i] (n_in, RC)."""
    prog = Program(plans)
    out = [None] * len(plans)
    for job in prog.jobs:
        pi = int(job["plan"][0])
        out[pi] = Emu(prog, job, RC).run([inputs[pi]], bwd)[0]
    return out, prog
