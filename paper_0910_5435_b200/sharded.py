"""Order-sharded SHT across GPUs: one process per GPU, one all-to-all per direction.

SURVEY.md §8(e): the orders m are independent — each |m| = mu owns its two
plans (even / odd degree chain) and the +-m pair shares them — so rank r keeps
the plans of a contiguous order range [mu_begin_r, mu_end_r) only, cut so that
every rank holds about the same butterfly storage.  The single exchange step
is the m <-> theta transpose between the Legendre stage (local orders, all 2l
latitudes) and the phi-DFT (all orders, a slab of latitudes):

  synthesis:  beta --Legendre(local mu)--> g[bins_r][b][all t]
              --all-to-all--> g[all bins][b][slab_r] --DFT over bins--> grid[b][slab_r][n]
  analysis:   grid[b][slab_r][n] --DFT--> G[all bins][b][slab_r]
              --all-to-all--> G[bins_r][b][all t] --Legendre^T(local mu)--> beta (local orders)

bins_r = {mu} U {N - mu : mu > 0} for mu in the rank's range (N = 4l - 1).  The
collective is ``torch.distributed.all_to_all_single`` on the float64 view of
the complex buffers (NCCL over NVLink on the GPUs; gloo in the CPU tests), with
uneven split sizes (alltoallv).  The phi-DFT here is torch.fft (cuFFT); the
Legendre stage is the CUDA engine through the C ABI (``SHT.range``).

The reference has no multi-process path; this module is the
host plumbing around the per-rank engine, mirroring ``SHT``'s entry points.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def dense_words(l: int, mu: int) -> int:
    """Words of the two dense chain matrices of order mu: l * (n_e + n_o) = l * (2l - mu)."""
    return l * (2 * l - mu)


def partition_orders(l: int, world: int, weights=None) -> list[tuple[int, int]]:
    """Contiguous order ranges [a, b) covering 0..2l-1, one per rank, with
    near-equal total weight (default: dense words per order; pass measured
    plan.stored_words per order to balance by butterfly storage).  Every rank
    gets at least one order when 2l >= world."""
    n = 2 * l
    if world < 1:
        raise ValueError("partition: world size must be >= 1")
    w = np.asarray(weights if weights is not None else [dense_words(l, mu) for mu in range(n)], dtype=np.float64)
    if w.shape != (n,) or np.any(w < 0):
        raise ValueError(f"partition: need {n} non-negative per-order weights")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        c = int(np.searchsorted(cum, target))
        if c > 0 and abs(cum[c - 1] - target) <= abs(cum[min(c, n)] - target):
            c -= 1
        lo = cuts[-1] + (1 if n - cuts[-1] > world - r else 0)  # leave >= 1 order per remaining rank
        hi = n - (world - r)
        cuts.append(int(min(max(c, lo), max(hi, lo))))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def latitude_slabs(l: int, world: int) -> list[tuple[int, int]]:
    """Rows [t0, t1) of the 2l-row grid per rank (as even as possible)."""
    rows = 2 * l
    base, extra = divmod(rows, world)
    out, t = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((t, t + n))
        t += n
    return out


def order_bins(l: int, mu_begin: int, mu_end: int) -> np.ndarray:
    """phi-stage bins of orders [mu_begin, mu_end): mu for +mu, N - mu for -mu (mu > 0)."""
    N = 4 * l - 1
    pos = list(range(mu_begin, mu_end))
    neg = [N - mu for mu in range(max(mu_begin, 1), mu_end)]
    return np.array(pos + neg, dtype=np.int64)


def coefficient_slices(l: int, mu_begin: int, mu_end: int) -> list[tuple[int, int]]:
    """[offset, offset + length) ranges of the packed coefficient vector held by an order range."""
    from .sht import coeff_offset
    out = []
    for mu in range(mu_begin, mu_end):
        for m in ((mu,) if mu == 0 else (mu, -mu)):
            o = coeff_offset(l, m)
            out.append((o, o + 2 * l - mu))
    return out


@dataclass
class ShardLayout:
    l: int
    world: int
    rank: int
    orders: list[tuple[int, int]]
    slabs: list[tuple[int, int]]

    @property
    def N(self) -> int:
        return 4 * self.l - 1

    def bins(self, r: int) -> np.ndarray:
        return order_bins(self.l, *self.orders[r])

    @property
    def my_orders(self) -> tuple[int, int]:
        return self.orders[self.rank]

    @property
    def my_slab(self) -> tuple[int, int]:
        return self.slabs[self.rank]


def exchange_tables(lay: "ShardLayout", batch: int):
    """Offsets of the fused sharded path (include/bfly_b200.h, bfly_sht_shard_*):
    order-side buffer (synthesis send / analysis receive): peer j's block holds
    [my bin][member][row of j's slab]; slab-side buffer (synthesis receive /
    analysis send): peer r's block holds [r's bin][member][row of my slab].
    Returns (row_base[2l], row_T[2l], bin_off[N], order_sizes[W], slab_sizes[W])
    with sizes in complex elements."""
    l, W, me = lay.l, lay.world, lay.rank
    n = [len(lay.bins(r)) for r in range(W)]
    T = [t1 - t0 for (t0, t1) in lay.slabs]
    order_sizes = [n[me] * batch * T[j] for j in range(W)]
    slab_sizes = [n[r] * batch * T[me] for r in range(W)]
    obase = np.concatenate([[0], np.cumsum(order_sizes)[:-1]]).astype(np.int64)
    sbase = np.concatenate([[0], np.cumsum(slab_sizes)[:-1]]).astype(np.int64)
    row_base = np.empty(2 * l, np.int64)
    row_T = np.empty(2 * l, np.int32)
    for j, (t0, t1) in enumerate(lay.slabs):
        row_base[t0:t1] = obase[j] + np.arange(t1 - t0)
        row_T[t0:t1] = T[j]
    bin_off = np.empty(lay.N, np.int64)
    for r in range(W):
        bins = lay.bins(r)
        bin_off[bins] = sbase[r] + np.arange(len(bins), dtype=np.int64) * batch * T[me]
    return row_base, row_T, bin_off, order_sizes, slab_sizes


def make_layout(l: int, world: int, rank: int, weights=None) -> ShardLayout:
    return ShardLayout(l, world, rank, partition_orders(l, world, weights), latitude_slabs(l, world))


class ShardedSHT:
    """SHT of bandlimit l sharded over the ranks of a torch.distributed group.

    legendre: the rank's Legendre engine for its order range — an ``SHT``
    built with ``SHT.range`` (CUDA, the product path) or any object with the
    same ``legendre_synthesize(beta, out)`` / ``legendre_analyze(gdft, out)``
    over the full (4l-1, B, 2l) bin layout.

    Data distribution: coefficients use the packed 4l^2 layout (only the
    rank's orders are read / written, the rest of an output is zero); the grid
    is the rank's latitude slab, shape (B, t1 - t0, 4l - 1).
    """

    def __init__(self, layout: ShardLayout, legendre, group=None):
        self.layout = layout
        self.legendre = legendre
        self.group = group
        self.l, self.N = layout.l, layout.N
        self._tables = {}  # batch -> device tables of the fused path

    def _fused(self) -> bool:
        """The CUDA engine of this library: parity combine / split and the slab
        DFT run fused on the device (bfly_sht_shard_*), no torch reshuffles."""
        import ctypes as C
        from ._lib import check, lib
        from .sht import SHT
        if not isinstance(self.legendre, SHT) or getattr(self.legendre, "mu_range", None) is None:
            return False
        if not hasattr(self, "_fused_ok"):
            ok = C.c_int(0)
            check(lib().bfly_sht_shard_supported(self.legendre._h, C.byref(ok)))
            self._fused_ok = bool(ok.value)
        return self._fused_ok

    def _device_tables(self, batch: int, device):
        import torch
        key = (batch, str(device))
        if key not in self._tables:
            rb, rt, bo, osz, ssz = exchange_tables(self.layout, batch)
            self._tables[key] = (torch.from_numpy(rb).to(device), torch.from_numpy(rt).to(device),
                                 torch.from_numpy(bo).to(device), osz, ssz)
        return self._tables[key]

    def _exchange(self, flat_in, sizes_in, sizes_out):
        """alltoallv of complex buffers (counts in complex elements) on the float64 view."""
        import torch
        import torch.distributed as dist
        if self.layout.world == 1:
            return flat_in  # one peer: the send buffer is the receive buffer
        out = torch.empty(sum(sizes_out), dtype=torch.complex128, device=flat_in.device)
        dist.all_to_all_single(torch.view_as_real(out).reshape(-1), torch.view_as_real(flat_in).reshape(-1),
                               [2 * c for c in sizes_out], [2 * c for c in sizes_in], group=self.group)
        return out

    def _stream(self, device):
        import torch
        return torch.cuda.current_stream(device).cuda_stream

    # -- the fused device steps either side of the exchange ---------------------
    # Each returns one flat complex128 buffer laid out as exchange_tables()
    # describes; the per-peer blocks are consecutive, so the buffer is the
    # alltoallv operand as is.
    def synth_pack(self, beta):
        """Legendre stage of the local orders + parity combine, written straight
        into the send buffer (bfly_sht_shard_synthesize)."""
        import ctypes as C
        import torch
        from ._lib import check, lib
        B = beta.shape[0]
        rb, rt, _, osz, _ = self._device_tables(B, beta.device)
        send = torch.empty(sum(osz), dtype=torch.complex128, device=beta.device)
        check(lib().bfly_sht_shard_synthesize(self.legendre._h, C.c_void_p(beta.data_ptr()),
                                              C.c_void_p(send.data_ptr()), C.c_void_p(rb.data_ptr()),
                                              C.c_void_p(rt.data_ptr()), B, C.c_void_p(self._stream(beta.device))))
        return send

    def synth_finish(self, recv, batch: int):
        """phi-DFT of the rank's latitude slab from the received bins (bfly_sht_shard_phi)."""
        import ctypes as C
        import torch
        from ._lib import check, lib
        _, _, bo, _, _ = self._device_tables(batch, recv.device)
        t0, t1 = self.layout.my_slab
        grid = torch.empty((batch, t1 - t0, self.N), dtype=torch.complex128, device=recv.device)
        check(lib().bfly_sht_shard_phi(self.legendre._h, 1, C.c_void_p(recv.data_ptr()), C.c_void_p(grid.data_ptr()),
                                       C.c_void_p(bo.data_ptr()), t1 - t0, batch,
                                       C.c_void_p(self._stream(recv.device))))
        return grid

    def anal_pack(self, grid_slab):
        """phi-DFT of the slab, bins scattered into the per-owner send blocks."""
        import ctypes as C
        import torch
        from ._lib import check, lib
        B = grid_slab.shape[0]
        _, _, bo, _, ssz = self._device_tables(B, grid_slab.device)
        t0, t1 = self.layout.my_slab
        g = grid_slab.contiguous()
        send = torch.empty(sum(ssz), dtype=torch.complex128, device=g.device)
        check(lib().bfly_sht_shard_phi(self.legendre._h, 0, C.c_void_p(g.data_ptr()), C.c_void_p(send.data_ptr()),
                                       C.c_void_p(bo.data_ptr()), t1 - t0, B, C.c_void_p(self._stream(g.device))))
        return send

    def anal_finish(self, recv, batch: int):
        """Parity split + transposed Legendre stage of the local orders (bfly_sht_shard_analyze)."""
        import ctypes as C
        import torch
        from ._lib import check, lib
        rb, rt, _, _, _ = self._device_tables(batch, recv.device)
        beta = torch.zeros((batch, 4 * self.l * self.l), dtype=torch.complex128, device=recv.device)
        check(lib().bfly_sht_shard_analyze(self.legendre._h, C.c_void_p(recv.data_ptr()), C.c_void_p(beta.data_ptr()),
                                           C.c_void_p(rb.data_ptr()), C.c_void_p(rt.data_ptr()), batch,
                                           C.c_void_p(self._stream(recv.device))))
        return beta

    @classmethod
    def create(cls, l: int, eps: float = 1e-12, group=None, device: int | None = None, weights=None,
               block_width: int = 60, threads: int | None = None) -> "ShardedSHT":
        import torch.distributed as dist
        from .sht import SHT
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        layout = make_layout(l, world, rank, weights)
        if device is None:
            import torch
            device = torch.cuda.current_device()
        eng = SHT.range(l, *layout.my_orders, eps=eps, block_width=block_width, threads=threads, device=device)
        return cls(layout, eng, group)

    # -- the exchange (alltoallv on the float64 view) ---------------------------
    def _all_to_all(self, send: list, recv_shapes: list):
        import torch
        import torch.distributed as dist
        sizes_in = [int(t.numel()) * 2 for t in send]
        sizes_out = [int(np.prod(s)) * 2 for s in recv_shapes]
        flat_in = torch.cat([torch.view_as_real(t.contiguous()).reshape(-1) for t in send])
        flat_out = torch.empty(sum(sizes_out), dtype=torch.float64, device=flat_in.device)
        if self.layout.world == 1:
            flat_out.copy_(flat_in)
        else:
            dist.all_to_all_single(flat_out, flat_in, sizes_out, sizes_in, group=self.group)
        out, o = [], 0
        for s, n in zip(recv_shapes, sizes_out):
            out.append(torch.view_as_complex(flat_out[o:o + n].view(*s, 2)))
            o += n
        return out

    def synthesize(self, beta):
        """beta (B, 4l^2), rank's orders filled -> the rank's grid slab (B, T, 4l-1)."""
        import torch
        lay = self.layout
        B = beta.shape[0]
        if self._fused():
            _, _, _, osz, ssz = self._device_tables(B, beta.device)
            return self.synth_finish(self._exchange(self.synth_pack(beta), osz, ssz), B)
        g = torch.zeros((self.N, B, 2 * self.l), dtype=torch.complex128, device=beta.device)
        self.legendre.legendre_synthesize(beta, out=g)
        mine = torch.as_tensor(lay.bins(lay.rank), device=beta.device)
        gl = g.index_select(0, mine)  # (n_r, B, 2l)
        send = [gl[:, :, t0:t1] for (t0, t1) in lay.slabs]
        t0, t1 = lay.my_slab
        recv = self._all_to_all(send, [(len(lay.bins(r)), B, t1 - t0) for r in range(lay.world)])
        full = torch.empty((self.N, B, t1 - t0), dtype=torch.complex128, device=beta.device)
        for r, part in enumerate(recv):
            full.index_copy_(0, torch.as_tensor(lay.bins(r), device=beta.device), part)
        grid = torch.fft.ifft(full, dim=0) * self.N  # sum_m g_m e^{+2 pi i m n / N}
        return grid.permute(1, 2, 0).contiguous()

    def analyze(self, grid_slab):
        """The rank's grid slab (B, T, 4l-1) -> beta (B, 4l^2), rank's orders filled (rest zero)."""
        import torch
        lay = self.layout
        B = grid_slab.shape[0]
        t0, t1 = lay.my_slab
        if tuple(grid_slab.shape[1:]) != (t1 - t0, self.N):
            raise ValueError(f"analyze: slab shape {tuple(grid_slab.shape)}, expected (B, {t1 - t0}, {self.N})")
        if self._fused():
            _, _, _, osz, ssz = self._device_tables(B, grid_slab.device)
            return self.anal_finish(self._exchange(self.anal_pack(grid_slab), ssz, osz), B)
        G = torch.fft.fft(grid_slab, dim=-1).permute(2, 0, 1)  # (N, B, T), unnormalised
        send = [G.index_select(0, torch.as_tensor(lay.bins(r), device=G.device)) for r in range(lay.world)]
        nb = len(lay.bins(lay.rank))
        recv = self._all_to_all(send, [(nb, B, s1 - s0) for (s0, s1) in lay.slabs])
        gfull = torch.zeros((self.N, B, 2 * self.l), dtype=torch.complex128, device=grid_slab.device)
        mine = torch.as_tensor(lay.bins(lay.rank), device=grid_slab.device)
        gl = torch.cat(recv, dim=2)  # slabs are consecutive row ranges
        gfull.index_copy_(0, mine, gl)
        beta = torch.zeros((B, 4 * self.l * self.l), dtype=torch.complex128, device=grid_slab.device)
        self.legendre.legendre_analyze(gfull, out=beta)
        return beta


# ---- the native sharded handle (C++ behind the C ABI, bfly_shard_*) ----------------
def native_layout(l: int, world: int):
    """(orders, slabs) as the C++ host layer computes them (bfly_shard_layout)."""
    import ctypes as C
    from ._lib import check, lib
    o = (C.c_int64 * (2 * world))()
    s = (C.c_int64 * (2 * world))()
    check(lib().bfly_shard_layout(l, world, o, s))
    return ([(int(o[2 * r]), int(o[2 * r + 1])) for r in range(world)],
            [(int(s[2 * r]), int(s[2 * r + 1])) for r in range(world)])


def native_tables(l: int, world: int, rank: int, batch: int):
    """exchange_tables() as the C++ host layer computes them (bfly_shard_tables)."""
    import ctypes as C
    from ._lib import check, lib
    N = 4 * l - 1
    rb = np.empty(2 * l, np.int64)
    rt = np.empty(2 * l, np.int32)
    bo = np.empty(N, np.int64)
    osz = np.empty(world, np.int64)
    ssz = np.empty(world, np.int64)
    p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    check(lib().bfly_shard_tables(l, world, rank, batch, p64(rb), rt.ctypes.data_as(C.POINTER(C.c_int32)), p64(bo),
                                  p64(osz), p64(ssz)))
    return rb, rt, bo, [int(x) for x in osz], [int(x) for x in ssz]


class NativeShardedSHT:
    """The order-sharded SHT run by the C++ host layer (bfly_shard_create /
    synthesize / analyze): the rank's plans, the NCCL group (loaded by the
    library at run time, world > 1), the pipelined alltoallv -- the same data
    distribution as ShardedSHT (packed coefficients of the rank's orders, the
    rank's latitude slab of the grid).  The NCCL unique id travels through the
    torch.distributed group when one is initialised."""

    def __init__(self, l: int, eps: float = 1e-12, device: int = 0, block_width: int = 60,
                 threads: int | None = None, rank: int | None = None, world: int | None = None, nccl_id=None):
        import ctypes as C
        import os
        from ._lib import BFLY_OK, lib
        if world is None or rank is None:
            try:
                import torch.distributed as dist
                init = dist.is_initialized()
            except Exception:  # noqa: BLE001
                init = False
            world = dist.get_world_size() if init else 1
            rank = dist.get_rank() if init else 0
        if world > 1 and nccl_id is None:
            import torch.distributed as dist
            buf = [None]
            if rank == 0:
                idb = (C.c_char * 128)()
                self._ck(lib().bfly_shard_nccl_id(idb))
                buf[0] = bytes(idb)
            dist.broadcast_object_list(buf, src=0)
            nccl_id = buf[0]
        idp = None
        if nccl_id is not None:
            self._id = (C.c_char * 128).from_buffer_copy(nccl_id)
            idp = C.cast(self._id, C.c_void_p)
        out = C.c_void_p()
        threads = threads or max(1, (os.cpu_count() or 1) // max(1, world))
        self._ck(lib().bfly_shard_create(l, float(eps), block_width, threads, rank, world, idp, device, C.byref(out)))
        self._h = out
        info = (C.c_int64 * 7)()
        self._ck(lib().bfly_shard_info(self._h, info))
        self.l, self.N, self.device, self.world, self.rank = l, 4 * l - 1, device, world, rank
        self.my_orders = (int(info[0]), int(info[1]))
        self.my_slab = (int(info[2]), int(info[3]))
        self.fused_phi = bool(info[6])
        del BFLY_OK

    def chunk(self, batch: int) -> int:
        """Members per pipeline chunk (the C++ rule, csrc/shard.cpp)."""
        import os
        env = int(os.environ.get("BFLY_SHARD_CHUNK", "0") or 0)
        if env > 0:
            return min(env, batch)
        if self.world == 1:
            return batch
        if batch >= 32:
            return 16
        if batch >= 4:
            return (batch + 1) // 2
        return batch

    def range_sht(self):
        """The rank's order-range SHT handle (owned by this object) as an SHT."""
        import ctypes as C
        from ._lib import lib
        from .sht import SHT
        h = C.c_void_p()
        self._ck(lib().bfly_shard_sht(self._h, C.byref(h)))
        s = SHT.__new__(SHT)
        s.l, s.N, s.device = self.l, self.N, self.device
        s._h = h
        s._borrowed = True
        s.mu_range = self.my_orders
        return s

    @staticmethod
    def _ck(rc: int):
        from ._lib import BflyError, lib
        if rc != 0:
            raise BflyError(rc, lib().bfly_shard_last_error().decode())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            from ._lib import lib
            lib().bfly_shard_destroy(h)
            self._h = None

    def _stream(self, t):
        import torch
        return torch.cuda.current_stream(t.device).cuda_stream

    def synthesize(self, beta, out=None):
        """beta (B, 4l^2) complex128 on the device (the rank's orders read) -> slab (B, T, 4l-1)."""
        import ctypes as C
        import torch
        from ._lib import lib
        B = beta.shape[0]
        t0, t1 = self.my_slab
        if out is None:
            out = torch.empty((B, t1 - t0, self.N), dtype=torch.complex128, device=beta.device)
        self._ck(lib().bfly_shard_synthesize(self._h, C.c_void_p(beta.data_ptr()), C.c_void_p(out.data_ptr()), B,
                                             C.c_void_p(self._stream(beta))))
        return out

    def analyze(self, grid_slab, out=None):
        """slab (B, T, 4l-1) -> beta (B, 4l^2): the rank's orders written (the rest untouched)."""
        import ctypes as C
        import torch
        from ._lib import lib
        B = grid_slab.shape[0]
        if out is None:
            out = torch.zeros((B, 4 * self.l * self.l), dtype=torch.complex128, device=grid_slab.device)
        self._ck(lib().bfly_shard_analyze(self._h, C.c_void_p(grid_slab.data_ptr()), C.c_void_p(out.data_ptr()), B,
                                          C.c_void_p(self._stream(grid_slab))))
        return out
