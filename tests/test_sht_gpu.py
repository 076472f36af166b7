"""Spherical harmonic transforms on the GPU vs the CPU oracle (oracle/sht_oracle.py).

Tolerance (north_star): relative l2 <= 1e-10 in fp64.  With the reference's
own plans and weights the engine must agree to <= 1e-12; with this library's
plans (its own, more accurate GL rule) to <= 1e-10.
"""
import os

import numpy as np
import pytest
import torch

import paper_0910_5435_b200 as bb
from oracle import sht_oracle

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module", params=[32, 256])
def pair(request, oracle):
    l = request.param
    ref = sht_oracle.RefSHT(l, 1e-12)
    plans = [bb.ButterflyPlan.from_bfly1(ref.plans.plan(i).save()) for i in range(len(ref.plans))]
    same = bb.SHT.from_plans(l, plans, rho=ref.rho)
    return l, ref, same


def test_synthesis_same_plans(pair):
    l, ref, sht = pair
    beta = sht_oracle.random_coefficients(l, 2, seed=1000 + l)
    got = sht.synthesize(torch.from_numpy(beta).cuda()).cpu().numpy()
    assert relerr(got, ref.synthesize(beta)) <= 1e-12


def test_analysis_same_plans(pair):
    l, ref, sht = pair
    beta = sht_oracle.random_coefficients(l, 2, seed=2000 + l)
    grid = ref.synthesize(beta)
    got = sht.analyze(torch.from_numpy(grid).cuda()).cpu().numpy()
    assert relerr(got, ref.analyze(grid)) <= 1e-12


def test_legendre_stage_same_plans(pair):
    l, ref, sht = pair
    beta = sht_oracle.random_coefficients(l, 1, seed=3000 + l)
    g = sht.legendre_synthesize(torch.from_numpy(beta).cuda()).cpu().numpy()  # [bin][b][t]
    g_ref, _ = ref.legendre_synthesis(beta)                                  # [b][t][bin]
    assert relerr(np.transpose(g, (1, 2, 0)), g_ref) <= 1e-12
    gd = np.fft.fft(ref.synthesize(beta), axis=-1)
    b_gpu = sht.legendre_analyze(torch.from_numpy(np.ascontiguousarray(np.transpose(gd, (2, 0, 1)))).cuda())
    b_ref, _ = ref.legendre_analysis(gd)
    assert relerr(b_gpu.cpu().numpy(), b_ref) <= 1e-12


def test_own_plans_vs_oracle_and_round_trip(pair):
    l, ref, _ = pair
    sht = bb.SHT(l, eps=1e-12)
    beta = sht_oracle.random_coefficients(l, 3, seed=4000 + l, decaying_member=2)
    tb = torch.from_numpy(beta).cuda()
    grid = sht.synthesize(tb)
    g_ref = ref.synthesize(beta)
    assert relerr(grid.cpu().numpy(), g_ref) <= 1e-10
    back = sht.analyze(grid).cpu().numpy()
    assert relerr(back, beta) <= 1e-10
    # decaying-spectrum member on its own (BASELINE.json config 3)
    assert relerr(back[2], beta[2]) <= 1e-10


def test_host_api_matches_device_api():
    l = 32
    sht = bb.SHT(l)
    beta = sht_oracle.random_coefficients(l, 2, seed=7)
    dev = sht.synthesize(torch.from_numpy(beta).cuda()).cpu().numpy()
    host = sht.synthesize_host(beta)
    assert np.array_equal(dev, host)
    assert np.array_equal(sht.analyze_host(host), sht.analyze(torch.from_numpy(host).cuda()).cpu().numpy())


@pytest.mark.parametrize("l", [1, 2, 3, 5, 8, 13, 32])
def test_independent_dense_check_small_l(l):
    """Smallest bandlimits (single-entry plans, N = 3, 7, 11, 19 (a generic radix), 31, 51, 127)
    against an independent scipy evaluation, both directions."""
    sht = bb.SHT(l, eps=1e-13)
    beta = sht_oracle.random_coefficients(l, 2, seed=11 + l)
    f = sht.synthesize_host(beta)
    fd = np.stack([sht_oracle.dense_synthesis(l, beta[b], sht.cos_theta()) for b in range(2)]).reshape(f.shape)
    assert relerr(f, fd) <= 1e-12
    assert relerr(sht.analyze_host(fd), beta) <= 1e-12


GOLD = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


@pytest.mark.parametrize("l", [16, 32])
def test_golden_fixtures(l):
    """Against outputs of the reference itself (tests/golden/make_golden.py); no oracle library needed."""
    g = np.load(f"{GOLD}/sht_l{l}.npz")
    sht = bb.SHT(l, eps=float(g["eps"]))
    grid = sht.synthesize(torch.from_numpy(g["beta"]).cuda()).cpu().numpy()
    assert relerr(grid, g["grid"]) <= 1e-10
    back = sht.analyze(torch.from_numpy(g["grid"]).cuda()).cpu().numpy()
    assert relerr(back, g["back"]) <= 1e-10
    assert relerr(back, g["beta"]) <= 1e-10


@pytest.mark.parametrize("waves", [False, True])
@pytest.mark.parametrize("l,cuts", [(32, [0, 9, 64]), (64, [0, 1, 40, 127, 128])])
def test_order_ranges_compose(l, cuts, waves, monkeypatch):
    """Shards of the order range (SHT.range) write disjoint bins / coefficients that
    sum to the full transform (whole-chain and wave programs)."""
    if waves:
        monkeypatch.setenv("BFLY_WAVES", "1")
    full = bb.SHT(l, eps=1e-12)
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, 2, seed=5000 + l)).cuda()
    g_full = full.legendre_synthesize(beta)
    gd = torch.fft.fft(full.synthesize(beta), dim=-1).permute(2, 0, 1).contiguous()
    b_full = full.legendre_analyze(gd)
    g_sum = torch.zeros_like(g_full)
    b_sum = torch.zeros_like(b_full)
    for a, b in zip(cuts[:-1], cuts[1:]):
        part = bb.SHT.range(l, a, b, eps=1e-12)
        g = torch.zeros_like(g_full)
        part.legendre_synthesize(beta, out=g)
        g_sum += g
        bt = torch.zeros_like(b_full)
        part.legendre_analyze(gd, out=bt)
        b_sum += bt
    assert relerr(g_sum.cpu().numpy(), g_full.cpu().numpy()) <= 1e-14
    assert relerr(b_sum.cpu().numpy(), b_full.cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("l,fused", [(32, True), (48, False)])
def test_sharded_single_rank_matches_full(l, fused):
    """l=48: N=191 is a prime above the in-kernel DFT's radix limit, so the
    sharded transform takes the Legendre-entry-point + cuFFT route."""
    sh = bb.ShardedSHT.create(l, eps=1e-12)
    assert sh._fused() == fused
    full = bb.SHT(l, eps=1e-12)
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, 2, seed=6000)).cuda()
    slab = sh.synthesize(beta)
    assert relerr(slab.cpu().numpy(), full.synthesize(beta).cpu().numpy()) <= 1e-13
    assert relerr(sh.analyze(slab).cpu().numpy(), beta.cpu().numpy()) <= 1e-10


@pytest.mark.parametrize("l,W,B,waves", [(32, 2, 2, False), (47, 3, 3, False), (64, 4, 1, False), (40, 5, 2, False),
                                          (64, 2, 5, True), (47, 3, 17, True)])
def test_sharded_fused_steps_emulated_ranks(l, W, B, waves, monkeypatch):
    """The fused sharded path (bfly_sht_shard_*) for W ranks, run one after another
    in this process: each rank's send buffer is cut into its per-peer blocks and
    the alltoallv is done by slicing (what NCCL moves between GPUs), then every
    rank's slab / coefficients are compared with the single-GPU transform and the
    oracle.  waves: every rank's Legendre stage on the wave programs."""
    from paper_0910_5435_b200.sharded import exchange_tables, make_layout
    full = bb.SHT(l, eps=1e-12)
    if waves:
        monkeypatch.setenv("BFLY_WAVES", "1")
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=6100 + W)).cuda()
    grid_full = full.synthesize(beta)
    ranks = []
    for r in range(W):
        lay = make_layout(l, W, r)
        ranks.append(bb.ShardedSHT(lay, bb.SHT.range(l, *lay.my_orders, eps=1e-12), None))
    assert all(sh._fused() for sh in ranks)

    def alltoallv(sends, send_sizes, recv_sizes):
        blocks = [list(torch.split(s, sz)) for s, sz in zip(sends, send_sizes)]
        out = []
        for r in range(W):
            parts = [blocks[j][r] for j in range(W)]
            assert [p.numel() for p in parts] == recv_sizes[r]
            out.append(torch.cat(parts))
        return out

    tabs = [exchange_tables(sh.layout, B) for sh in ranks]
    sends = [sh.synth_pack(beta) for sh in ranks]
    recvs = alltoallv(sends, [t[3] for t in tabs], [t[4] for t in tabs])
    slabs = [sh.synth_finish(rv, B) for sh, rv in zip(ranks, recvs)]
    for sh, slab in zip(ranks, slabs):
        t0, t1 = sh.layout.my_slab
        assert relerr(slab.cpu().numpy(), grid_full[:, t0:t1].cpu().numpy()) <= 1e-13
    sends = [sh.anal_pack(slab) for sh, slab in zip(ranks, slabs)]
    recvs = alltoallv(sends, [t[4] for t in tabs], [t[3] for t in tabs])
    beta_sum = sum(sh.anal_finish(rv, B) for sh, rv in zip(ranks, recvs))
    assert relerr(beta_sum.cpu().numpy(), beta.cpu().numpy()) <= 1e-10
    assert relerr(beta_sum.cpu().numpy(), full.analyze(grid_full).cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("waves", ["1", "0"])
@pytest.mark.parametrize("l,B", [(1024, 16)])
def test_full_size_round_trip(l, B, waves, monkeypatch):
    """BASELINE.json configs[2] at full size (l=1024, 16 functions, one with a
    (k+1)^-2 spectrum): size-independent properties of the exact transform pair —
    analysis(synthesis(beta)) = beta, and linearity — on the wave programs (the
    default at this size) and on the whole-chain engine."""
    monkeypatch.setenv("BFLY_WAVES", waves)
    sht = bb.SHT(l, eps=1e-12)
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=7000, decaying_member=B - 1)).cuda()
    grid = sht.synthesize(beta)
    back = sht.analyze(grid)
    err = (torch.linalg.vector_norm(back - beta) / torch.linalg.vector_norm(beta)).item()
    assert err <= 1e-10
    # the decaying member on its own (its norm is tiny next to the others)
    d = B - 1
    err_d = (torch.linalg.vector_norm(back[d] - beta[d]) / torch.linalg.vector_norm(beta[d])).item()
    assert err_d <= 1e-10
    # linearity: synth(a x + y) = a synth(x) + synth(y)
    g2 = sht.synthesize(2.5 * beta[:2] + beta[2:4])
    lin = (torch.linalg.vector_norm(g2 - (2.5 * grid[:2] + grid[2:4])) / torch.linalg.vector_norm(g2)).item()
    assert lin <= 1e-13
    # N = 4095 rows run the large-row phi kernels; the same program through the
    # stage-wise cuFFT route (program cache reload) gives the same transforms
    assert sht.info()["l"] == l
    import os
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "c3.bin")
        sht.save(path)
        os.environ["BFLY_PHI"] = "cufft"
        try:
            ref = bb.SHT.load(path)
        finally:
            del os.environ["BFLY_PHI"]
    g_ref = ref.synthesize(beta[:3])
    assert relerr(grid[:3].cpu().numpy(), g_ref.cpu().numpy()) <= 1e-14
    b_ref = ref.analyze(grid[:3])
    assert relerr(back[:3].cpu().numpy(), b_ref.cpu().numpy()) <= 1e-14
    # real fields at this size (three-buffer real phi kernels)
    n = l * (2 * l + 1)
    half = bb.half_from_full(l, beta[:2].cpu().numpy())
    half[:, :2 * l] = half[:, :2 * l].real
    g_cplx = sht.synthesize(torch.from_numpy(bb.full_from_half(l, half)).cuda())
    g_real = sht.synthesize_real(torch.from_numpy(half).cuda())
    assert g_real.shape == (2, 2 * l, 4 * l - 1) and half.shape == (2, n)
    assert relerr(g_real.cpu().numpy(), g_cplx.real.cpu().numpy()) <= 1e-13
    assert relerr(sht.analyze_real(g_real).cpu().numpy(), half) <= 1e-10


@pytest.mark.parametrize("l", [32, 64, 100])
def test_phi_large_row_kernels(l, monkeypatch):
    """The large-row phi kernels (one row at a time per CTA, 3 N complex of shared
    memory; default from l ~ 900) forced at small l agree with the two-row kernels."""
    sht = bb.SHT(l, eps=1e-12)
    monkeypatch.setenv("BFLY_PHI_BIG", "1")
    big = bb.SHT(l, eps=1e-12)
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, 3, seed=6300 + l)).cuda()
    g = sht.synthesize(beta)
    gb = big.synthesize(beta)
    assert relerr(gb.cpu().numpy(), g.cpu().numpy()) <= 1e-14
    assert relerr(big.analyze(g).cpu().numpy(), sht.analyze(g).cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("l,bw,B", [(32, 60, 1), (64, 60, 2), (96, 60, 3), (200, 60, 17), (300, 160, 5), (256, 60, 16)])
def test_wave_programs(l, bw, B, monkeypatch, tmp_path):
    """Level-synchronous wave programs (every StripeId of a level for all 4B
    right-hand sides per launch on the FP64 tensor cores, roots on the batched
    root kernels) agree with the whole-chain program in both directions, and the
    round trip holds, including >64 right-hand sides (two column chunks), tall
    dense stripes and ranks above 128."""
    whole = bb.SHT(l, eps=1e-12, block_width=bw)
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=6500 + l, decaying_member=B - 1)).cuda()
    g0 = whole.synthesize(beta)
    b0 = whole.analyze(g0)
    monkeypatch.setenv("BFLY_WAVES", "1")
    wv = bb.SHT(l, eps=1e-12, block_width=bw)
    assert wv.info()["stored_words"] == whole.info()["stored_words"]
    g = wv.synthesize(beta)
    b = wv.analyze(g0)
    assert relerr(g.cpu().numpy(), g0.cpu().numpy()) <= 1e-13
    assert relerr(b.cpu().numpy(), b0.cpu().numpy()) <= 1e-13
    assert relerr(wv.analyze(g).cpu().numpy(), beta.cpu().numpy()) <= 1e-10
    # real fields (half-layout coefficients, two fields per 4-column slot); they
    # need the fused phi stage (4l - 1 without prime factors above 127)
    half = bb.half_from_full(l, beta.cpu().numpy())
    half[:, :2 * l] = half[:, :2 * l].real
    hb = torch.from_numpy(half).cuda()
    try:
        gr = whole.synthesize_real(hb)
    except bb.BflyInvalidArgument:
        gr = None
    if gr is not None:
        assert relerr(wv.synthesize_real(hb).cpu().numpy(), gr.cpu().numpy()) <= 1e-13
        assert relerr(wv.analyze_real(gr).cpu().numpy(), half) <= 1e-10
    # the stage-wise entry points (Legendre stage alone, [bin][b][t] layout)
    gl = wv.legendre_synthesize(beta)
    assert relerr(gl.cpu().numpy(), whole.legendre_synthesize(beta).cpu().numpy()) <= 1e-13
    assert relerr(wv.legendre_analyze(gl).cpu().numpy(), whole.legendre_analyze(gl).cpu().numpy()) <= 1e-13
    # program cache: a reloaded wave program gives bit-identical transforms
    path = str(tmp_path / "w.bin")
    wv.save(path)
    re = bb.SHT.load(path)
    assert re.info()["stored_words"] == wv.info()["stored_words"]
    assert torch.equal(re.synthesize(beta), g) and torch.equal(re.analyze(g0), b)


@pytest.mark.parametrize("l,B", [(1, 1), (2, 3), (3, 2), (5, 4), (8, 9), (13, 33)])
def test_wave_programs_small_bandlimits(l, B, monkeypatch):
    """Wave programs at the smallest bandlimits (single-leaf dense plans: every
    chain is one full-rank leaf feeding its root through a copy node; the empty odd
    chain of mu = 2l - 1; the mu = 0 -m half) against the independent dense SHT, with
    batches that exercise the 8 / 16 / 32 / 64-column tiles and a tail chunk."""
    monkeypatch.setenv("BFLY_WAVES", "1")
    wv = bb.SHT(l, eps=1e-12)
    assert wv.program_info()["waves"] == 1 and wv.program_info()["whole"] == 0
    beta = sht_oracle.random_coefficients(l, B, seed=6800 + l)
    g = wv.synthesize(torch.from_numpy(beta).cuda()).cpu().numpy()
    gd = np.stack([sht_oracle.dense_synthesis(l, beta[b], wv.cos_theta()) for b in range(B)]).reshape(g.shape)
    assert relerr(g, gd) <= 1e-12
    back = wv.analyze(torch.from_numpy(g).cuda()).cpu().numpy()
    assert relerr(back, beta) <= 1e-12


def test_both_programs_dispatch_by_batch(monkeypatch):
    """BFLY_WAVES=2 (the default from l = 512): one handle holds the whole-chain
    and the wave programs and picks per call by batch size (waves from
    BFLY_WAVE_MIN_BATCH functions on); both routes give the same transforms, and
    the program cache keeps both."""
    l = 64
    monkeypatch.setenv("BFLY_WAVES", "0")
    whole = bb.SHT(l, eps=1e-12)
    monkeypatch.setenv("BFLY_WAVES", "2")
    monkeypatch.setenv("BFLY_WAVE_MIN_BATCH", "3")
    both = bb.SHT(l, eps=1e-12)
    for B in (1, 2, 3, 6):
        beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=6600 + B)).cuda()
        g = both.synthesize(beta)
        assert relerr(g.cpu().numpy(), whole.synthesize(beta).cpu().numpy()) <= 1e-13
        assert relerr(both.analyze(g).cpu().numpy(), beta.cpu().numpy()) <= 1e-10
    import tempfile, os
    with tempfile.TemporaryDirectory() as d:
        both.save(os.path.join(d, "p.bin"))
        re = bb.SHT.load(os.path.join(d, "p.bin"))
    for B in (1, 6):
        beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=6700 + B)).cuda()
        assert torch.equal(re.synthesize(beta), both.synthesize(beta))


@pytest.mark.parametrize("l,bw,B", [(64, 60, 1), (96, 60, 3), (200, 60, 17), (300, 160, 5)])
def test_split_root_kernels(l, bw, B, monkeypatch):
    """Split programs (event program + separate root stage) with each root
    stage — the batched FP64 tensor-core kernels (default, cell-major C / partial
    rows, all 4B right-hand sides per skeleton read), the per-member
    matrix-vector kernels and engine root jobs — agree with the whole-chain
    program.  Covers more than 64 right-hand sides (B = 17: two column chunks),
    stripes taller than one 128-row block (dense high-order plans, l = 200, 300)
    and ranks above 128 (block width 160)."""
    whole = bb.SHT(l, eps=1e-12, block_width=bw)
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=6400 + l, decaying_member=B - 1)).cuda()
    g0 = whole.synthesize(beta)
    b0 = whole.analyze(g0)
    monkeypatch.setenv("BFLY_SPLIT", "1")
    for roots in ("mma", "rootmv", "engine"):
        monkeypatch.setenv("BFLY_ROOTS", roots)
        sp = bb.SHT(l, eps=1e-12, block_width=bw)
        g = sp.synthesize(beta)
        b = sp.analyze(g0)
        assert relerr(g.cpu().numpy(), g0.cpu().numpy()) <= 1e-13, roots
        assert relerr(b.cpu().numpy(), b0.cpu().numpy()) <= 1e-13, roots
    assert relerr(b0.cpu().numpy(), beta.cpu().numpy()) <= 1e-10


@pytest.mark.parametrize("l,split", [(64, False), (48, False), (64, True), (64, "waves")])
def test_batch_chunking_bit_identical(l, split, monkeypatch):
    """Full transforms run large batches as member chunks when their scratch
    exceeds BFLY_SCRATCH_GB; chunked and unchunked results agree — bit for bit on
    the fused path, to rounding where cuFFT plans for another batch count may
    pick other kernels (l=48, split programs)."""
    if split == "waves":
        monkeypatch.setenv("BFLY_WAVES", "1")
    elif split:
        monkeypatch.setenv("BFLY_SPLIT", "1")
    sht = bb.SHT(l, eps=1e-12)
    B = 5
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=6200 + l)).cuda()
    g1 = sht.synthesize(beta)
    b1 = sht.analyze(g1)
    per_member = 32.0 * sht.info()["n_plans"] * l
    monkeypatch.setenv("BFLY_SCRATCH_GB", repr(2.5 * per_member / 1e9))  # chunks of <= 2 members
    g2 = sht.synthesize(beta)
    b2 = sht.analyze(g1)
    monkeypatch.setenv("BFLY_SCRATCH_GB", "1e-12")  # one member at a time
    g3 = sht.synthesize(beta)
    if l == 64 and split is False:
        assert torch.equal(g1, g2) and torch.equal(b1, b2) and torch.equal(g1, g3)
    else:
        for x, y in ((g2, g1), (b2, b1), (g3, g1)):
            assert relerr(x.cpu().numpy(), y.cpu().numpy()) <= 1e-14
    assert relerr(b1.cpu().numpy(), beta.cpu().numpy()) <= 1e-10


def test_host_api_pinned_buffers():
    """The host-buffer entry points on pinned memory (the bench's e2e path)."""
    l = 64
    sht = bb.SHT(l, eps=1e-12)
    beta = sht_oracle.random_coefficients(l, 2, seed=8000)
    want = sht.synthesize(torch.from_numpy(beta).cuda()).cpu().numpy()
    beta_h = torch.from_numpy(beta).pin_memory()
    grid_h = torch.empty((2, 2 * l, 4 * l - 1), dtype=torch.complex128).pin_memory()
    back_h = torch.empty_like(beta_h).pin_memory()
    sht.synthesize_host_ptr(beta_h.data_ptr(), grid_h.data_ptr(), 2)
    assert relerr(grid_h.numpy(), want) <= 1e-15
    sht.analyze_host_ptr(grid_h.data_ptr(), back_h.data_ptr(), 2)
    assert relerr(back_h.numpy(), beta) <= 1e-10


def test_sharded_over_nccl_single_rank():
    """The order-sharded transform through a real NCCL process group (one rank on
    this box; the multi-rank exchange is covered with gloo in tests/test_sharded.py)."""
    import os
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29600 + os.getpid() % 1000))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        l = 32
        sh = bb.ShardedSHT.create(l, eps=1e-12, device=0)
        beta = torch.from_numpy(sht_oracle.random_coefficients(l, 3, seed=9000, decaying_member=2)).cuda()
        slab = sh.synthesize(beta)
        ref = sht_oracle.RefSHT(l, 1e-12).synthesize(beta.cpu().numpy())
        assert relerr(slab.cpu().numpy(), ref) <= 1e-10
        assert relerr(sh.analyze(slab).cpu().numpy(), beta.cpu().numpy()) <= 1e-10
    finally:
        if own:
            dist.destroy_process_group()


def test_argument_errors():
    """Reference-style error behaviour at the boundary (std::invalid_argument <-> BflyInvalidArgument)."""
    import ctypes as C
    from paper_0910_5435_b200._lib import check, lib
    l = 8
    sht = bb.SHT(l)
    with pytest.raises(ValueError):
        sht.synthesize(torch.zeros((1, 4 * l * l - 1), dtype=torch.complex128, device="cuda"))
    with pytest.raises(TypeError):
        sht.synthesize(torch.zeros((1, 4 * l * l), dtype=torch.complex64, device="cuda"))
    beta = torch.zeros((1, 4 * l * l), dtype=torch.complex128, device="cuda")
    grid = torch.empty((1, 2 * l, 4 * l - 1), dtype=torch.complex128, device="cuda")
    with pytest.raises(bb.BflyInvalidArgument):
        check(lib().bfly_sht_synthesize(sht._h, C.c_void_p(beta.data_ptr()), C.c_void_p(grid.data_ptr()), 0, None))
    part = bb.SHT.range(l, 0, 4)
    with pytest.raises(bb.BflyInvalidArgument, match="partial order range"):
        part.synthesize(beta)
    # zero in, exactly zero out (reference tests/test_butterfly.cpp:135-141)
    assert torch.count_nonzero(sht.synthesize(beta)).item() == 0


def test_program_cache_round_trip(tmp_path):
    """the packed device program saved and reloaded without
    rebuilding plans gives bit-identical transforms."""
    l = 64
    sht = bb.SHT(l, eps=1e-12)
    path = str(tmp_path / "sht64.bflysht")
    sht.save(path)
    again = bb.SHT.load(path)
    assert again.info()["stored_words"] == sht.info()["stored_words"]
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, 2, seed=9100)).cuda()
    g1, g2 = sht.synthesize(beta), again.synthesize(beta)
    assert torch.equal(g1, g2)
    assert torch.equal(sht.analyze(g1), again.analyze(g1))
    with open(path, "r+b") as f:
        f.write(b"NOTASHT!")
    with pytest.raises(bb.BflySerializationError):
        bb.SHT.load(path)


@pytest.mark.parametrize("l,B", [(8, 1), (8, 3), (32, 2), (256, 1), (256, 4)])
def test_real_field_transforms(l, B):
    """Real fields (one field: RC = 2 engine; several: two fields per task on the
    four right-hand sides) and the shared-DFT phi kernels agree with the complex
    transform of the Hermitian-symmetric coefficients."""
    sht = bb.SHT(l, eps=1e-12)
    rng = np.random.default_rng(9200 + l + B)
    n = l * (2 * l + 1)
    half = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    half[:, :2 * l] = half[:, :2 * l].real  # Im beta^0 = 0
    full = bb.full_from_half(l, half)
    g_cplx = sht.synthesize(torch.from_numpy(full).cuda())
    assert torch.max(torch.abs(g_cplx.imag)).item() <= 1e-10 * torch.max(torch.abs(g_cplx.real)).item()
    g_real = sht.synthesize_real(torch.from_numpy(half).cuda())
    assert relerr(g_real.cpu().numpy(), g_cplx.real.cpu().numpy()) <= 1e-13
    back = sht.analyze_real(g_real).cpu().numpy()
    assert relerr(back, half) <= 1e-10
    assert np.array_equal(bb.half_from_full(l, full), half)


@pytest.mark.parametrize("l,force", [(2, True), (3, True), (5, True), (8, True), (32, True), (33, False)])
def test_rader_prime_rows(l, force, monkeypatch):
    """Prime N = 4l - 1 through Rader's algorithm (phi_rader.cu: in-place DIF /
    DIT convolution of length N - 1): forced at small primes (7, 11, 19, 31,
    127) against the Stockham kernels, and by default above the Stockham radix
    limit (l = 33: N = 131) against the scipy dense synthesis, both directions."""
    if force:
        monkeypatch.setenv("BFLY_PHI_RADER", "1")
    sht = bb.SHT(l, eps=1e-13)
    beta = sht_oracle.random_coefficients(l, 3, seed=8100 + l)
    tb = torch.from_numpy(beta).cuda()
    g = sht.synthesize(tb)
    back = sht.analyze(g)
    assert relerr(back.cpu().numpy(), beta) <= 1e-12
    if force:
        monkeypatch.delenv("BFLY_PHI_RADER")
        ref = bb.SHT(l, eps=1e-13)
        assert relerr(g.cpu().numpy(), ref.synthesize(tb).cpu().numpy()) <= 1e-13
        assert relerr(back.cpu().numpy(), ref.analyze(g).cpu().numpy()) <= 1e-13
    else:
        fd = np.stack([sht_oracle.dense_synthesis(l, beta[b], sht.cos_theta()) for b in range(3)])
        assert relerr(g.cpu().numpy(), fd.reshape(g.shape)) <= 1e-12
        assert relerr(sht.analyze(torch.from_numpy(fd.reshape(g.shape)).cuda()).cpu().numpy(), beta) <= 1e-12


def test_out_argument_validation():
    """A caller-supplied out= must match what the kernels write."""
    sht = bb.SHT(8)
    beta = torch.from_numpy(sht_oracle.random_coefficients(8, 2, seed=3)).cuda()
    with pytest.raises(ValueError):
        sht.synthesize(beta, out=torch.empty((1, 16, 31), dtype=torch.complex128, device="cuda"))
    with pytest.raises(TypeError):
        sht.synthesize(beta, out=torch.empty((2, 16, 31), dtype=torch.complex64, device="cuda"))
    grid = sht.synthesize(beta)
    with pytest.raises(ValueError):
        sht.analyze(grid, out=torch.empty((2, 255), dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):
        sht.legendre_synthesize(beta, out=torch.empty((31, 1, 16), dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):
        sht.analyze(grid, out=torch.empty((2, 256), dtype=torch.complex128, device="cuda").t().contiguous().t())


@pytest.mark.parametrize("l,bw,B", [(64, 60, 2), (96, 60, 3), (200, 60, 17), (300, 160, 5), (256, 60, 16),
                                    (512, 250, 3)])
def test_graph_program_groups_and_engine(l, bw, B, monkeypatch):
    """The graph program (one persistent, dependency-ordered launch per
    direction, wgraph.cu) with small plan groups (many groups in flight at
    once) against the default grouping (bit-identical: the queue order does
    not change any sum) and the whole-chain engine (one function at a time);
    column blocks of 8 / 16 / 32 with partial blocks (R = 4B = 8, 12, 68, 20,
    64, 12), ranks and root stripes above the 192-row pass (block width 250 at
    l = 512), repeated launches (the per-launch epoch of the completion flags)."""
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=7100 + l, decaying_member=B - 1)).cuda()
    monkeypatch.setenv("BFLY_WAVES", "2")
    monkeypatch.setenv("BFLY_WAVE_MIN_BATCH", "1")
    ref = bb.SHT(l, eps=1e-12, block_width=bw)
    monkeypatch.setenv("BFLY_GRAPH_GROUP", "64")
    gr = bb.SHT(l, eps=1e-12, block_width=bw)
    assert gr.program_info()["graph_groups"] > ref.program_info()["graph_groups"] >= 1
    g0 = ref.synthesize(beta)
    g1 = gr.synthesize(beta)
    assert torch.equal(g1, g0)
    b0 = ref.analyze(g0)
    assert torch.equal(gr.analyze(g0), b0)
    assert relerr(gr.analyze(g1).cpu().numpy(), beta.cpu().numpy()) <= 1e-10
    for _ in range(3):
        assert torch.equal(gr.synthesize(beta), g1)
    # the wavefront queue order (diagonals over the small groups): another topological order of the
    # same items, bit-identical results
    monkeypatch.setenv("BFLY_GRAPH_WAVEFRONT", "1")
    wf = bb.SHT(l, eps=1e-12, block_width=bw)
    monkeypatch.delenv("BFLY_GRAPH_WAVEFRONT")
    assert torch.equal(wf.synthesize(beta), g0)
    assert torch.equal(wf.analyze(g0), b0)
    del wf
    # the whole-chain engine, one function per call (where it exists)
    if ref.program_info()["whole"]:
        monkeypatch.setenv("BFLY_WAVE_MIN_BATCH", "1000")
        eng = bb.SHT(l, eps=1e-12, block_width=bw)
        assert not eng.uses_waves(B)
        ge = eng.synthesize(beta)
        assert relerr(g1.cpu().numpy(), ge.cpu().numpy()) <= 1e-13
        assert relerr(gr.analyze(g0).cpu().numpy(), eng.analyze(g0).cpu().numpy()) <= 1e-13
    gl = gr.legendre_synthesize(beta)
    assert relerr(gl.cpu().numpy(), ref.legendre_synthesize(beta).cpu().numpy()) <= 1e-14
    assert relerr(gr.legendre_analyze(gl).cpu().numpy(), ref.legendre_analyze(gl).cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("l,B", [(64, 4), (48, 3), (256, 5), (128, 33)])
def test_native_shard_single_rank(l, B, monkeypatch):
    """The C++ sharded handle (bfly_shard_*: own plan build, pipelined member
    chunks on two streams, the fused slab DFT or -- l = 48, N = 191 -- cuFFT on
    the slab rows) with one rank against the single-GPU transform."""
    from paper_0910_5435_b200.sharded import NativeShardedSHT
    monkeypatch.setenv("BFLY_SHARD_CHUNK", "2")
    sh = NativeShardedSHT(l, eps=1e-12, world=1, rank=0)
    assert sh.my_orders == (0, 2 * l) and sh.my_slab == (0, 2 * l)
    assert sh.fused_phi == (l != 48)
    full = bb.SHT(l, eps=1e-12)
    beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=8200 + l)).cuda()
    g = sh.synthesize(beta)
    g0 = full.synthesize(beta)
    assert relerr(g.cpu().numpy(), g0.cpu().numpy()) <= 1e-13
    b = sh.analyze(g0)
    assert relerr(b.cpu().numpy(), full.analyze(g0).cpu().numpy()) <= 1e-13
    assert relerr(sh.analyze(g).cpu().numpy(), beta.cpu().numpy()) <= 1e-10


def test_streamed_order_shards_round_trip(tmp_path):
    """scripts/c5_streamed.py (c5 on one GPU: the order shards one after the
    other into one exchange buffer) at a small bandlimit: round trip and the
    sampled orders against the reference."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "c5.json"
    subprocess.run([sys.executable, os.path.join(root, "scripts", "c5_streamed.py"), "--l", "96", "--batch", "8",
                    "--shards", "3", "--oracle", "--out", str(out)], check=True, cwd=root)
    res = json.loads(out.read_text())
    assert res["round_trip_rel_l2"] <= 1e-10, res
    assert max(res["round_trip_rel_l2_per_member"]) <= 1e-10, res
    assert max(res["oracle_rel_l2"].values()) <= 1e-10, res
