#!/usr/bin/env python
"""Benchmark: spherical-harmonic transform pairs (synthesis + analysis) per second.

Metric (BASELINE.json): "SHT pairs/sec (fwd+inv) vs bandlimit l; achieved HBM
GB/s / roofline fraction".  BASELINE.json's metric names no configuration, so
the default workload is the largest one that fits one GPU: configs[3] (c4,
l = 2048, 64 functions, fp64 complex N(0,1) coefficients, grid 4096 x 8191,
ID precision 1e-12); c1-c3 and c4 at eps 1e-10 are selectable.  A step is one
synthesis + one analysis of the batch on device-resident data; L2 is flushed
(256 MiB write) before every timed step and the flush is outside the step's
events (c3/c4 inputs are also far larger than L2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
    python bench.py --impl reference ...      # the reference CPU path, same workload

Multi-GPU (torchrun, one rank per GPU): each rank transforms its own batch
(weak scaling, no data-path collective); the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import numpy as np
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SHT pairs/sec (fwd+inv)"
UNIT = "pairs/s"

# Workloads (BASELINE.json configs).  The headline (default) is c4, the largest
# configuration that fits one GPU; c1-c3 stay selectable (--config).
CONFIGS = {
    "c1": dict(l=32, batch=1, eps=1e-12,
               text="configs[0]: l=32, 1 function, grid 64x127, eps 1e-12"),
    "c2": dict(l=256, batch=1, eps=1e-12,
               text="configs[1]: l=256, 1 function, grid 512x1023, eps 1e-12"),
    "c3": dict(l=1024, batch=16, eps=1e-12, decaying=15,
               text="configs[2]: l=1024, batch 16 (member 15 scaled by (k+1)^-2), grid 2048x4095, eps 1e-12"),
    "c4": dict(l=2048, batch=64, eps=1e-12,
               text="configs[3]: l=2048, batch 64, grid 4096x8191, eps 1e-12 (the eps 1e-10 plan set: "
                    "--config c4e10)"),
    "c4e10": dict(l=2048, batch=64, eps=1e-10,
                  text="configs[3]: l=2048, batch 64, grid 4096x8191, eps 1e-10"),
    # c5's plan set (~0.2 TB) does not fit one GPU: sharded runs only (torchrun, >= 2 ranks); on one
    # GPU scripts/c5_streamed.py runs the shards one after the other
    "c5": dict(l=4096, batch=8, eps=1e-12, min_gpus=2,
               text="configs[4]: l=4096, batch 8, grid 8192x16383, eps 1e-12, orders sharded over the GPUs"),
}
DEFAULT_CONFIG = "c4"
# Orders at or above this bandlimit: the CPU reference is timed on a strided
# sample of the orders and scaled to all of them (the full reference transform
# takes CPU-minutes to CPU-hours there).
CPU_SAMPLE_MIN_L = 1024
CPU_SAMPLE_ORDERS = 32


def fp64_peak():
    """Measured FP64 tensor-core (DMMA) and FMA peaks of this B200
    (scripts/fp64_peak.cu -> profiles/r02_fp64_peak.json): the roofline
    denominator of the batched Legendre stage (MEASURED_PEAKS.json has no FP64
    figure).  Falls back to the B200 spec sheet (40 TF/s) if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")) as f:
            p = json.load(f)
        tf = max(p["dmma_m8n8k4_tflops"], p["dmma_m16n8k16_tflops"], p["dfma_tflops"])
        return tf, "measured (scripts/fp64_peak.cu, profiles/r02_fp64_peak.json: max of DMMA and DFMA)"
    except Exception:
        return 40.0, "fallback: B200 spec FP64 tensor-core peak"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons, polled through NVML every ~2 ms in a
    background thread while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None
        self.nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        self._stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm = [m for m, _ in self.samples]
        reasons = sorted({name for _, rs in self.samples for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def sampled_orders(l: int) -> list[int]:
    """Every order below CPU_SAMPLE_MIN_L; above it a strided sample (unbiased
    for the sum over orders, whose cost falls with mu)."""
    if l < CPU_SAMPLE_MIN_L:
        return list(range(2 * l))
    stride = 2 * l // CPU_SAMPLE_ORDERS
    return list(range(stride // 2, 2 * l, stride))


class CpuReference:
    """The reference CPU path on one function of the workload: bfly::apply /
    apply_transpose (oracle/_ref = the unmodified reference sources) on the
    GL-row plans of the sampled orders, one vector per call, a std::thread pool
    over plans; plus the numpy phi DFT over the whole grid.  Per pair:
    t = t_legendre(sample) * (2l / orders sampled) + t_phi."""

    def __init__(self, cfg, nthreads: int):
        from oracle import ref, sht_oracle
        self.l = l = cfg["l"]
        self.orders = sampled_orders(l)
        self.nthreads = nthreads
        t0 = time.perf_counter()
        if len(self.orders) == 2 * l:
            self.shts = [sht_oracle.RefSHT(l, cfg["eps"], nthreads=nthreads)]
        else:  # per-order plan sets, built concurrently (the ctypes calls release the GIL)
            from concurrent.futures import ThreadPoolExecutor

            def one(mu):
                return sht_oracle.RefSHT(l, cfg["eps"], nthreads=2,
                                         planset=ref.RefPlanSet(l, cfg["eps"], mu_range=(mu, mu + 1), nthreads=2))
            with ThreadPoolExecutor(max_workers=max(1, min(nthreads, len(self.orders)))) as ex:
                self.shts = list(ex.map(one, self.orders))
        self.build_s = time.perf_counter() - t0
        self.scale = 2 * l / len(self.orders)
        self.beta = sht_oracle.random_coefficients(l, 1, seed=1000)
        self.sht_oracle = sht_oracle

    def _one(self, r, inner):
        r.nthreads = inner
        g = r.legendre_synthesis_bins(self.beta)
        r.legendre_analysis_bins(g, self.back)

    def legendre_pass(self, nthreads=None) -> float:
        """One synthesis + analysis of the sampled orders; seconds.  With a
        sample, the per-order plan sets run concurrently (the ctypes calls
        release the GIL), two plans each, so all threads stay busy."""
        from concurrent.futures import ThreadPoolExecutor
        nt = nthreads or self.nthreads
        self.back = np.zeros_like(self.beta)
        t0 = time.perf_counter()
        if len(self.shts) == 1:
            self._one(self.shts[0], nt)
        elif nt == 1:
            for r in self.shts:
                self._one(r, 1)
        else:
            with ThreadPoolExecutor(max_workers=min(nt, len(self.shts))) as ex:
                list(ex.map(lambda r: self._one(r, 2), self.shts))
        return time.perf_counter() - t0

    def phi_pass(self, nthreads=None) -> float:
        """Inverse + forward DFT of one function's full grid (2l x (4l-1)),
        scipy.fft (pocketfft) with one worker per thread."""
        import scipy.fft as sfft
        l = self.l
        nt = nthreads or self.nthreads
        g = np.random.default_rng(5).standard_normal((2 * l, 4 * l - 1)) + 0j
        t0 = time.perf_counter()
        f = sfft.ifft(g, axis=-1, workers=nt)
        sfft.fft(f, axis=-1, workers=nt)
        return time.perf_counter() - t0

    def pairs_per_s(self, seconds: float, min_passes: int = 2, nthreads=None):
        self.legendre_pass(nthreads)  # warm-up
        n, el = 0, 0.0
        while n < min_passes or el < seconds:
            el += self.legendre_pass(nthreads)
            n += 1
        t_phi = min(self.phi_pass(nthreads) for _ in range(3))
        t_pair = el / n * self.scale + t_phi
        return 1.0 / t_pair, n, el, t_phi

    def sample_text(self, n, el, cores) -> str:
        l = self.l
        if len(self.orders) == 2 * l:
            what = f"all {2 * l} orders"
        else:
            what = (f"{len(self.orders)} of {2 * l} orders (every {2 * l // len(self.orders)}th from "
                    f"{self.orders[0]}; Legendre time scaled by {self.scale:.0f})")
        return (f"{n} synthesis+analysis passes of one l={l} function over {what} in {el:.1f} s: reference "
                f"bfly::apply / apply_transpose (oracle/_ref, unmodified sources), one vector per call, "
                f"{cores} thread(s) over plans; scipy.fft phi stage on the full grid ({cores} worker(s))")


def cpu_baseline(args, cfg) -> dict:
    """The reference CPU path on a bounded sample of the workload, all host
    threads and one (the line's cpu_baseline)."""
    ncores = os.cpu_count() or 1
    try:
        cr = CpuReference(cfg, ncores)
        v, n, el, t_phi = cr.pairs_per_s(args.cpu_seconds)
        v1, n1, el1, _ = cr.pairs_per_s(min(args.cpu_seconds, 10.0), min_passes=1, nthreads=1)
        out = {"value": v, "unit": UNIT, "cores": ncores, "kind": "reference",
               "sample": cr.sample_text(n, el, ncores), "plan_build_s": cr.build_s,
               "phi_s_per_pair": t_phi,
               "one_core": {"value": v1, "unit": UNIT, "cores": 1, "sample": cr.sample_text(n1, el1, 1)}}
        del cr
        return out
    except Exception as exc:  # the baseline is reported, never required
        return {"value": None, "unit": UNIT, "cores": ncores, "kind": "reference",
                "sample": f"unavailable: {exc}"}


def run_reference(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nthreads = os.cpu_count() or 1
    cr = CpuReference(cfg, nthreads)
    for _ in range(args.warmup):
        cr.legendre_pass()
    t_phi = min(cr.phi_pass() for _ in range(3))
    # a step = passes over the sampled orders until >= 0.5 s have gone by (the reference's own timing
    # rule, tools/bfly_main.cpp:48-60: warm-up, then repetitions up to a minimum time), so that a small
    # --steps does not time thread start-up instead of the apply
    # (the time of a pass is what legendre_pass measures: the applies, not the allocation of its output
    # buffer -- the same accounting as cpu_baseline)
    passes, el = 0, 0.0
    for _ in range(args.steps):
        ts = 0.0
        while ts < 0.5:
            ts += cr.legendre_pass()
            passes += 1
        el += ts
    t_pair = el / passes * cr.scale + t_phi  # one function
    value = 1.0 / t_pair
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_pair,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "reference",
                         "sample": cr.sample_text(passes, el, nthreads), "plan_build_s": cr.build_s},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, cfg, world):
    return {"workload": f"{args.config}: {cfg['text']}", "l": cfg["l"], "batch_per_gpu": cfg["batch"],
            "global_batch": cfg["batch"] * world, "eps": cfg["eps"], "block_width": 60,
            "grid": [2 * cfg["l"], 4 * cfg["l"] - 1], "parallelism": f"replicas{world}",
            "l2": "flushed before every timed step (256 MiB write, outside the step events)"}


def run_ours(args, cfg):
    import numpy as np
    import torch

    import paper_0910_5435_b200 as bb
    from oracle import sht_oracle  # only for the seeded input generator and the CPU baseline

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    l, B, eps = cfg["l"], cfg["batch"], cfg["eps"]
    N = 4 * l - 1
    nthreads = max(1, (os.cpu_count() or 1) // max(1, world))

    t0 = time.perf_counter()
    sht = bb.SHT(l, eps=eps, threads=nthreads, device=local)
    t_build = time.perf_counter() - t0
    info = sht.info()

    # seeded N(0,1) coefficients, generated member by member straight into the
    # pinned host buffer (member b: seed 1000 + 100 rank + b; the decaying
    # member of c3 scaled by (k+1)^-2)
    beta_pinned = torch.empty((B, 4 * l * l), dtype=torch.complex128, pin_memory=True)
    for b in range(B):
        dec = 0 if cfg.get("decaying") == b else None
        beta_pinned[b] = torch.from_numpy(
            sht_oracle.random_coefficients(l, 1, seed=1000 + 100 * rank + b, decaying_member=dec)[0])
    beta = beta_pinned.to(dev)
    grid = torch.empty((B, 2 * l, N), dtype=torch.complex128, device=dev)
    beta_out = torch.empty_like(beta)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():  # the public device API: coefficients -> grid -> coefficients
        sht.synthesize(beta, out=grid)
        sht.analyze(grid, out=beta_out)

    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    # correctness of the benchmarked pipeline: the round trip must reproduce beta
    rt = float((torch.linalg.vector_norm(beta_out - beta) / torch.linalg.vector_norm(beta)).item())
    if not rt <= 1e-9:
        raise SystemExit(f"bench: the benchmarked pipeline does not round-trip (rel l2 {rt:.3e}); refusing to report")

    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    sampler = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    sampler.start()
    # Timed region 1 (the headline value): K steps of the public API, nothing
    # but the step between the events (the launches stay back to back, so the
    # programmatic dependent launches between engine and phi kernels act).
    for k in range(K):
        flush.fill_(k & 0xFF)
        e = ev[k]
        e[0].record()
        sht.synthesize(beta, out=grid)
        e[1].record()
        sht.analyze(grid, out=beta_out)
        e[2].record()
    torch.cuda.synchronize()
    barrier(world)
    # Timed region 2 (the roofline): the same K steps with CUDA events around
    # every engine launch on its stream (which serialises the phi kernels).
    sht.engine_time(True)
    for k in range(K):
        flush.fill_(k & 0xFF)
        sht.synthesize(beta, out=grid)
        sht.analyze(grid, out=beta_out)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    eng_ms, eng_n = sht.engine_time(False)

    t_step = sum(e[0].elapsed_time(e[2]) for e in ev) / K  # ms
    t_syn = sum(e[0].elapsed_time(e[1]) for e in ev) / K
    t_ana = sum(e[1].elapsed_time(e[2]) for e in ev) / K
    t_step = allreduce_max(t_step, world)
    t_syn = allreduce_max(t_syn, world)
    t_ana = allreduce_max(t_ana, world)
    t_eng = [eng_ms[d] / max(1, eng_n[d]) for d in range(2)]  # ms per engine launch
    t_leg = [eng_ms[d] / K for d in range(2)]  # ms of Legendre stage per direction per step
    chunks = max(1, eng_n[0] // K)  # member chunks per call (large batches)
    value = world * B / (t_step * 1e-3)

    # Roofline of the Legendre stage: per direction, matrix
    # words read once + complex coefficients and grid bins read/written once;
    # FLOPs 2 R per matrix word (R = 4 B right-hand sides).
    bytes_l = 8 * info["stored_words"] + 16 * B * (4 * l * l + 2 * l * N)
    flops_l = 2 * 4 * B * info["stored_words"]  # R = 4 real RHS per function (mu = 0: 2, padded)
    t_kernel = allreduce_max(0.5 * (t_eng[0] + t_eng[1]), world) * 1e-3
    hbm, peak_kind = peaks()
    waves = sht.uses_waves(B)
    pinfo = sht.program_info()
    traffic = traffic_detail = None
    prof = os.path.join(ROOT, "profiles", f"ncu_engine_{args.config}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            pj = json.load(f)
        traffic = pj.get("dram_bytes_per_launch")
        traffic_detail = {k: pj[k] for k in ("dram_bytes_per_graph_launch", "member_chunks_per_direction", "source")
                          if k in pj} or None
    if not waves:
        # one function: the whole-chain engine, HBM bound (0.94 flop/B at c2)
        achieved = bytes_l / t_kernel / 1e9 if t_kernel > 0 else None  # None: no engine launch was timed
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm if achieved else None, "traffic": traffic, "peak_kind": peak_kind,
                    "kernel": "engine_kernel (butterfly apply, both directions)",
                    "algorithmic_bytes_per_launch": bytes_l, "flops_per_launch": flops_l,
                    "fetched_bytes_per_launch": info["fetched_bytes"]}
        launches = 4  # per step: engine + fused phi kernel, each direction
    else:
        # a batch: the wave programs (levels + roots on FP64 DMMA), tensor bound
        # (2 R flop per 8-byte word: 16 flop/B at R = 64); "launch" = the
        # Legendre stage of one direction (all its level / root launches)
        # per direction and step: all chunks' level / root launches
        t_dir = allreduce_max(0.5 * (t_leg[0] + t_leg[1]), world) * 1e-3
        achieved = flops_l / t_dir / 1e12 if t_dir > 0 else None
        peak_tf, peak_kind_tf = fp64_peak()
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": achieved / peak_tf if achieved else None, "traffic": traffic,
                    "peak_kind": peak_kind_tf,
                    "kernel": "wgraph_kernel (the graph program: every node and root block of one direction in one "
                              "persistent FP64 DMMA launch per member chunk): the Legendre stage of one direction for the "
                              "whole batch, event-timed per step",
                    "algorithmic_bytes_per_launch": bytes_l, "flops_per_launch": flops_l,
                    "legendre_ms_per_direction": [t_leg[0], t_leg[1]], "member_chunks": chunks,
                    "traffic_detail": traffic_detail,
                    "hbm_achieved_gbs": bytes_l / t_dir / 1e9 if t_dir > 0 else None}
        # per chunk: synthesis = coefficient gather + levels + one root launch per
        # root group + phi; analysis = phi + roots + levels + scatter
        if pinfo["graph"]:  # gather + graph + phi, phi + graph + scatter
            launches = chunks * 6
        else:
            launches = chunks * ((1 + pinfo["levels"] + pinfo["root_groups"] + 1) + (1 + 1 + pinfo["levels"] + 1))

    print(json.dumps({"device_step_ms": t_step, "legendre_ms": t_leg, "value": value, "build_s": t_build}),
          file=sys.stderr, flush=True)
    # the device-resident tensors go before the host path allocates its own staging
    del beta, grid, beta_out, flush
    torch.cuda.empty_cache()
    # End to end through the C ABI with pinned host buffers (copies inside the timed region).
    # The analysis writes the coefficients back into the input buffer (c4: 17 GB
    # of coefficients + 34 GB of grid pinned).
    beta_h = beta_pinned
    grid_h = torch.empty((B, 2 * l, N), dtype=torch.complex128, pin_memory=True)
    back_h = beta_h
    for _ in range(max(1, args.warmup)):
        sht.synthesize_host_ptr(beta_h.data_ptr(), grid_h.data_ptr(), B)
        sht.analyze_host_ptr(grid_h.data_ptr(), back_h.data_ptr(), B)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(K):
        sht.synthesize_host_ptr(beta_h.data_ptr(), grid_h.data_ptr(), B)
        sht.analyze_host_ptr(grid_h.data_ptr(), back_h.data_ptr(), B)
    t_e2e = (time.perf_counter() - t0) / K
    barrier(world)
    t_e2e = allreduce_max(t_e2e, world)
    e2e_value = world * B / t_e2e
    coeff_bytes = 16 * B * 4 * l * l
    grid_bytes = 16 * B * 2 * l * N

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_block(args, cfg, world),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": coeff_bytes + grid_bytes,
                    "d2h_bytes_per_step": grid_bytes + coeff_bytes,
                    "path": "bfly_sht_synthesize_host + bfly_sht_analyze_host (pinned host buffers)",
                    "ms_per_step": 1e3 * t_e2e},
            "gpu_launches": launches * K,
            "program": "waves (batched, FP64 DMMA)" if waves else "whole-chain engine",
            "clocks": clocks,
            "stages_ms": {"synthesis": t_syn, "analysis": t_ana, "engine_synthesis": t_eng[0],
                          "engine_analysis": t_eng[1], "engine_launches_timed": sum(eng_n),
                          "legendre_synthesis_per_step": t_leg[0], "legendre_analysis_per_step": t_leg[1]},
            "plan": {"stored_words": info["stored_words"], "fetched_bytes": info["fetched_bytes"],
                     "n_plans": info["n_plans"], "n_jobs": info["n_jobs"], "smem_bytes": info["smem_bytes"],
                     "build_s": t_build},
            "round_trip_rel_l2": rt,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sharded(args, cfg):
    """Order-sharded transform through the C++ host layer
    (bfly_shard_*): every rank builds and holds the plans of its order range
    and a latitude slab of the grid; the m <-> theta transpose is a grouped
    ncclSend / ncclRecv alltoallv overlapped with the next member chunk.  The B
    functions are shared by all ranks, so the job size is fixed as N grows
    (strong scaling)."""
    import numpy as np
    import torch

    from oracle import sht_oracle  # seeded input generator (and the CPU baseline) only
    from paper_0910_5435_b200.sharded import NativeShardedSHT, coefficient_slices
    from paper_0910_5435_b200.sht import SHT

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    l, B, eps = cfg["l"], cfg["batch"], cfg["eps"]
    N = 4 * l - 1
    nthreads = max(1, (os.cpu_count() or 1) // max(1, world))
    t0 = time.perf_counter()
    sh = NativeShardedSHT(l, eps=eps, device=local, threads=nthreads)
    t_build = time.perf_counter() - t0
    mu0, mu1 = sh.my_orders
    s0, s1 = sh.my_slab
    segs = coefficient_slices(l, mu0, mu1)
    c0, c1 = segs[0][0], segs[-1][1]  # the rank's orders are one contiguous run of the packed vector
    # seeded N(0,1) coefficients of this rank's orders (member b: seed 1000 + b), pinned host copy
    host_in = torch.zeros((B, c1 - c0), dtype=torch.complex128, pin_memory=True)
    for b in range(B):
        dec = 0 if cfg.get("decaying") == b else None
        full = sht_oracle.random_coefficients(l, 1, seed=1000 + b, decaying_member=dec)[0]
        host_in[b] = torch.from_numpy(full[c0:c1])
    beta = torch.zeros((B, 4 * l * l), dtype=torch.complex128, device=dev)
    beta[:, c0:c1] = host_in.to(dev)
    back = torch.zeros_like(beta)
    slab = torch.empty((B, s1 - s0, N), dtype=torch.complex128, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        sh.synthesize(beta, out=slab)
        sh.analyze(slab, out=back)
    torch.cuda.synchronize()
    rt = float((torch.linalg.vector_norm(back[:, c0:c1] - beta[:, c0:c1]) /
                torch.linalg.vector_norm(beta[:, c0:c1])).item())
    rt = allreduce_max(rt, world)
    if not rt <= 1e-9:
        raise SystemExit(f"bench: the sharded pipeline does not round-trip (rel l2 {rt:.3e}); refusing to report")
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    sampler = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    sampler.start()
    for k in range(K):
        flush.fill_(k & 0xFF)
        ev[k][0].record()
        sh.synthesize(beta, out=slab)
        ev[k][1].record()
        sh.analyze(slab, out=back)
        ev[k][2].record()
    torch.cuda.synchronize()
    barrier(world)
    # the rank's Legendre stage (graph program) timed per direction for the roofline
    rsht = sh.range_sht()
    rsht.engine_time(True)
    for k in range(K):
        flush.fill_(k & 0xFF)
        sh.synthesize(beta, out=slab)
        sh.analyze(slab, out=back)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    eng_ms, _ = rsht.engine_time(False)
    t_step = allreduce_max(sum(e[0].elapsed_time(e[2]) for e in ev) / K, world)
    t_syn = allreduce_max(sum(e[0].elapsed_time(e[1]) for e in ev) / K, world)
    t_ana = allreduce_max(sum(e[1].elapsed_time(e[2]) for e in ev) / K, world)
    info = rsht.info()
    flops_local = 2 * 4 * B * info["stored_words"]
    t_dir = 0.5 * (eng_ms[0] + eng_ms[1]) / K * 1e-3
    achieved = flops_local / t_dir / 1e12 if t_dir > 0 else None
    peak_tf, peak_kind_tf = fp64_peak()

    # end to end: the rank's coefficients H2D from pinned memory, its slab and its
    # coefficients D2H, every step
    host_slab = torch.empty((B, s1 - s0, N), dtype=torch.complex128, pin_memory=True)
    host_out = torch.empty_like(host_in, pin_memory=True)
    for _ in range(max(1, args.warmup)):
        beta[:, c0:c1].copy_(host_in, non_blocking=True)
        sh.synthesize(beta, out=slab)
        host_slab.copy_(slab, non_blocking=True)
        sh.analyze(slab, out=back)
        host_out.copy_(back[:, c0:c1], non_blocking=True)
    torch.cuda.synchronize()
    barrier(world)
    te = time.perf_counter()
    for _ in range(K):
        beta[:, c0:c1].copy_(host_in, non_blocking=True)
        sh.synthesize(beta, out=slab)
        host_slab.copy_(slab, non_blocking=True)
        sh.analyze(slab, out=back)
        host_out.copy_(back[:, c0:c1], non_blocking=True)
    torch.cuda.synchronize()
    t_e2e = allreduce_max((time.perf_counter() - te) / K, world)
    bytes_in = allreduce_max(float(host_in.numel() * 16), world)
    bytes_out = allreduce_max(float((host_slab.numel() + host_out.numel()) * 16), world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg)
    chunks = -(-B // sh.chunk(B))
    if rank == 0:
        line = {
            "metric": METRIC, "value": B / (t_step * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_block(args, cfg, 1), global_batch=B,
                           parallelism=f"orders sharded over {world} rank(s) (C++ host layer, bfly_shard_*), "
                                       "NCCL grouped send/recv m<->theta transpose overlapped with the next member "
                                       "chunk"),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf if achieved else None, "traffic": None, "peak_kind": peak_kind_tf,
                         "kernel": "wgraph_kernel: rank 0's Legendre stage (its order range), one direction, "
                                   "event-timed per step",
                         "flops_per_launch": flops_local,
                         "legendre_ms_per_direction": [eng_ms[0] / K, eng_ms[1] / K]},
            "cpu_baseline": cpu,
            "e2e": {"value": B / t_e2e, "unit": UNIT, "h2d_bytes_per_step": bytes_in, "d2h_bytes_per_step": bytes_out,
                    "path": "per rank: its coefficients H2D (pinned), bfly_shard_synthesize + bfly_shard_analyze, "
                            "its grid slab and coefficients D2H; max over ranks", "ms_per_step": 1e3 * t_e2e},
            "gpu_launches": 8 * chunks * K, "clocks": clocks, "mode": "sharded",
            "stages_ms": {"synthesis": t_syn, "analysis": t_ana},
            "shard": {"orders_rank0": [mu0, mu1], "slab_rank0": [s0, s1], "fused_slab_dft": sh.fused_phi,
                      "member_chunk": sh.chunk(B)},
            "plan_build_s": t_build, "round_trip_rel_l2": rt,
        }
        print(json.dumps(line), flush=True)
    del sh
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    # NCCL's version banner goes to stdout, which must carry exactly one JSON line
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=DEFAULT_CONFIG)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", choices=["auto", "replicas", "sharded"], default="auto",
                    help="auto: one GPU -> the single-GPU transform, several -> sharded; "
                         "sharded: the orders of one batch are split over the GPUs (strong scaling, "
                         "C++ host layer + NCCL); replicas: each GPU transforms its own batch (weak scaling)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl != "reference" and world < cfg.get("min_gpus", 1):
        raise SystemExit(f"bench: --config {args.config} needs at least {cfg['min_gpus']} GPUs (its plan set does not fit "
                         "one); launch with torchrun, or run scripts/c5_streamed.py on one GPU")
    if args.impl != "reference" and world >= 2 and cfg.get("min_gpus", 1) > 1 and args.mode == "replicas":
        raise SystemExit(f"bench: --config {args.config} runs sharded only")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.mode == "sharded" or (args.mode == "auto" and int(os.environ.get("WORLD_SIZE", "1")) > 1):
        run_sharded(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
