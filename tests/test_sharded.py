"""Order-sharded SHT (paper_0910_5435_b200/sharded.py) on CPU ranks over gloo.

The exchange logic — order partition, latitude slabs, the alltoallv of the
m <-> theta transpose in both directions, the phi-DFT on a slab — runs in
world_size 2 and 3 process groups with the reference (oracle) Legendre stage
standing in for each rank's CUDA engine; the assembled result must equal the
single-process reference SHT.  The GPU Legendre stage of an order range is
checked in tests/test_sht_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0910_5435_b200.sharded import (ShardedSHT, coefficient_slices, latitude_slabs, make_layout,
                                          order_bins, partition_orders)


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


class OracleLegendre:
    """Test stand-in for a rank's engine: reference plans of one order range."""

    def __init__(self, l, mu0, mu1, eps=1e-12):
        from oracle import ref
        from oracle.sht_oracle import RefSHT
        self.sht = RefSHT(l, eps, planset=ref.RefPlanSet(l, eps, mu_range=(mu0, mu1), nthreads=1))

    def legendre_synthesize(self, beta, out):
        g, _ = self.sht.legendre_synthesis(beta.numpy())  # (B, 2l, N)
        out.copy_(torch.from_numpy(np.ascontiguousarray(g.transpose(2, 0, 1))))

    def legendre_analyze(self, gdft, out):
        beta, _ = self.sht.legendre_analysis(gdft.numpy().transpose(1, 2, 0))
        out.copy_(torch.from_numpy(beta))


def test_partition_covers_and_balances():
    for l, world in ((8, 1), (8, 2), (16, 3), (256, 8), (1024, 8), (4, 8)):
        parts = partition_orders(l, world)
        assert parts[0][0] == 0 and parts[-1][1] == 2 * l
        assert all(a < b for a, b in parts) and all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
        if 2 * l >= 8 * world:
            w = [sum(l * (2 * l - mu) for mu in range(a, b)) for a, b in parts]
            assert max(w) / min(w) < 1.1
    # measured weights move the cuts
    w = np.ones(32)
    w[:4] = 100
    assert partition_orders(16, 2, w)[0][1] <= 4
    with pytest.raises(ValueError):
        partition_orders(8, 2, np.ones(5))


def test_bins_and_slabs():
    l = 8
    N = 4 * l - 1
    allb = np.concatenate([order_bins(l, a, b) for a, b in partition_orders(l, 3)])
    assert sorted(allb.tolist()) == list(range(N))
    assert latitude_slabs(l, 3) == [(0, 6), (6, 11), (11, 16)]
    sl = [s for a, b in partition_orders(l, 3) for s in coefficient_slices(l, a, b)]
    cover = np.zeros(4 * l * l, int)
    for a, b in sl:
        cover[a:b] += 1
    assert np.all(cover == 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, l, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.sht_oracle import random_coefficients
        lay = make_layout(l, world, rank)
        sht = ShardedSHT(lay, OracleLegendre(l, *lay.my_orders))
        beta = random_coefficients(l, 2, 77, decaying_member=1)
        mine = np.zeros_like(beta)
        for a, b in coefficient_slices(l, *lay.my_orders):
            mine[:, a:b] = beta[:, a:b]
        slab = sht.synthesize(torch.from_numpy(mine))
        back = sht.analyze(slab)
        q.put((rank, lay.my_slab, lay.my_orders, slab.numpy(), back.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_round_trip_gloo(oracle, world):
    from oracle.sht_oracle import RefSHT, random_coefficients
    l = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, l, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    beta = random_coefficients(l, 2, 77, decaying_member=1)
    grid = RefSHT(l, 1e-12).synthesize(beta)
    back = np.zeros_like(beta)
    for rank, (t0, t1), (a, b), slab, bk in sorted(res, key=lambda r: r[0]):
        assert relerr(slab, grid[:, t0:t1]) <= 1e-13
        for o0, o1 in coefficient_slices(l, a, b):
            back[:, o0:o1] = bk[:, o0:o1]
    assert relerr(back, beta) <= 1e-12


@pytest.mark.parametrize("l,world", [(4, 1), (8, 3), (16, 5), (32, 8), (100, 7), (1024, 8), (2048, 8), (4096, 8)])
def test_native_layout_matches_python(l, world):
    """The C++ host layer's partition, slabs and exchange tables (bfly_shard_layout
    / bfly_shard_tables) equal sharded.py's, rank by rank."""
    from paper_0910_5435_b200 import sharded as sh
    orders, slabs = sh.native_layout(l, world)
    assert orders == sh.partition_orders(l, world)
    assert slabs == sh.latitude_slabs(l, world)
    if l <= 128:
        lay_all = [sh.make_layout(l, world, r) for r in range(world)]
        for r in range(world):
            for batch in (1, 3):
                want = sh.exchange_tables(lay_all[r], batch)
                got = sh.native_tables(l, world, r, batch)
                for a, b in zip(got[:3], want[:3]):
                    np.testing.assert_array_equal(a, b)
                assert got[3] == [int(x) for x in want[3]] and got[4] == [int(x) for x in want[4]]
