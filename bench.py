#!/usr/bin/env python
"""Benchmark: spherical-harmonic transform pairs (synthesis + analysis) per second.

Metric (BASELINE.json): "SHT pairs/sec (fwd+inv) vs bandlimit l; achieved HBM
GB/s / roofline fraction".  Default workload = BASELINE.json configs[1]
(l = 256, one function, fp64 complex N(0,1) coefficients, grid 512 x 1023,
ID precision 1e-12).  A step is one synthesis + one analysis of the batch on
device-resident data; L2 is flushed (256 MiB write) before every timed step
and the flush is outside the step's events.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
    python bench.py --impl reference ...      # the reference CPU path, same workload

Multi-GPU (torchrun, one rank per GPU): each rank transforms its own batch
(weak scaling, no data-path collective); the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SHT pairs/sec (fwd+inv)"
# FP64 tensor-core (DMMA) peak of this B200 at 1965 MHz, measured: ncu reports
# sm__ops_path_tensor_src_fp64 = 27.9 TF/s at 76.9 % DMMA-pipe activity
# (profiles/r01_c3_waves_ncu_summary.md); the B200 spec sheet says 40.
FP64_TENSOR_TFLOPS = 36.3
UNIT = "pairs/s"

CONFIGS = {
    "c1": dict(l=32, batch=1, eps=1e-12,
               text="configs[0]: l=32, 1 function, grid 64x127, eps 1e-12"),
    "c2": dict(l=256, batch=1, eps=1e-12,
               text="configs[1]: l=256, 1 function, grid 512x1023, eps 1e-12"),
    "c3": dict(l=1024, batch=16, eps=1e-12, decaying=15,
               text="configs[2]: l=1024, batch 16 (member 15 scaled by (k+1)^-2), grid 2048x4095, eps 1e-12"),
}


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


def cpu_reference_pairs(cfg, seconds: float, min_pairs: int, nthreads: int):
    """Reference CPU path on a bounded sample: (pairs/s, pairs, wall seconds, build seconds)."""
    from oracle import sht_oracle
    l, B = cfg["l"], cfg["batch"]
    t0 = time.perf_counter()
    ref = sht_oracle.RefSHT(l, cfg["eps"], nthreads=nthreads)
    t_build = time.perf_counter() - t0
    # one function per CPU step: the sample is a bounded slice of the batch
    beta = sht_oracle.random_coefficients(l, 1, seed=1000)
    grid = ref.synthesize(beta)  # warm-up
    ref.analyze(grid)
    n = 0
    t0 = time.perf_counter()
    while True:
        grid = ref.synthesize(beta)
        ref.analyze(grid)
        n += 1
        el = time.perf_counter() - t0
        if n >= min_pairs and el >= seconds:
            break
    return n / el, n, el, t_build


def run_reference(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nthreads = os.cpu_count() or 1
    from oracle import sht_oracle
    l = cfg["l"]
    t0 = time.perf_counter()
    ref = sht_oracle.RefSHT(l, cfg["eps"], nthreads=nthreads)
    t_build = time.perf_counter() - t0
    beta = sht_oracle.random_coefficients(l, 1, seed=1000)
    for _ in range(args.warmup):
        ref.analyze(ref.synthesize(beta))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.analyze(ref.synthesize(beta))
    el = time.perf_counter() - t0
    value = args.steps / el  # one function per step
    sample = (f"{args.steps} pairs of one l={l} function (reference bfly::apply / apply_transpose on every "
              f"GL-row plan, one vector per call, std::thread pool over plans; numpy FFT phi stage)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "reference",
                         "sample": sample, "plan_build_s": t_build},
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

    beta_np = sht_oracle.random_coefficients(l, B, seed=1000 + 100 * rank, decaying_member=cfg.get("decaying"))
    beta = torch.from_numpy(beta_np).to(dev)
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
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_engine_{args.config}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
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
        achieved = flops_l / t_kernel / 1e12 if t_kernel > 0 else None
        peak_tf = FP64_TENSOR_TFLOPS
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": achieved / peak_tf if achieved else None, "traffic": traffic,
                    "peak_kind": "measured: ncu DMMA-pipe peak (MEASURED_PEAKS.json has no FP64 figure; spec 40 TF/s)",
                    "kernel": "wave_fwd/wave_bwd + root_mma (Legendre stage per direction, FP64 DMMA)",
                    "algorithmic_bytes_per_launch": bytes_l, "flops_per_launch": flops_l,
                    "hbm_achieved_gbs": bytes_l / t_kernel / 1e9 if t_kernel > 0 else None}
        # synthesis: coefficient gather + levels + one root launch per root group +
        # phi; analysis: phi + roots + levels + scatter
        launches = (1 + pinfo["levels"] + pinfo["root_groups"] + 1) + (1 + 1 + pinfo["levels"] + 1)

    # End to end through the C ABI with pinned host buffers (copies inside the timed region).
    beta_h = torch.empty((B, 4 * l * l), dtype=torch.complex128, pin_memory=True)
    beta_h.copy_(torch.from_numpy(beta_np))
    grid_h = torch.empty((B, 2 * l, N), dtype=torch.complex128, pin_memory=True)
    back_h = torch.empty_like(beta_h, pin_memory=True)
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
        try:
            v, n, el, tb = cpu_reference_pairs(cfg, args.cpu_seconds, 3, os.cpu_count() or 1)
            cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "reference",
                   "sample": f"{n} pairs of one l={l} function in {el:.1f} s: reference bfly::apply / "
                             f"apply_transpose (oracle/_ref, unmodified sources) on all {info['n_plans']} "
                             f"GL-row plans, one vector per call, std::thread pool over plans; numpy FFT",
                   "plan_build_s": tb}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_block(args, cfg, world),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": coeff_bytes + grid_bytes,
                    "d2h_bytes_per_step": grid_bytes + coeff_bytes,
                    "path": "bfly_sht_synthesize_host + bfly_sht_analyze_host (pinned host buffers)"},
            "gpu_launches": launches * K,
            "program": "waves (batched, FP64 DMMA)" if waves else "whole-chain engine",
            "clocks": clocks,
            "stages_ms": {"synthesis": t_syn, "analysis": t_ana, "engine_synthesis": t_eng[0],
                          "engine_analysis": t_eng[1], "engine_launches_timed": sum(eng_n)},
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
    """Order-sharded transform: every rank holds the plans of
    its order range and a latitude slab of the grid; the m <-> theta transpose
    is an NCCL all-to-all.  The B functions are shared by all ranks, so the
    job size is fixed as N grows (strong scaling)."""
    import numpy as np
    import torch

    import paper_0910_5435_b200 as bb
    from oracle import sht_oracle  # seeded input generator only

    world, rank, local = dist_setup()
    if world > 1:
        pass
    else:  # a one-rank group so the collective path is the same code
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + (os.getpid() % 1000)))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    l, B, eps = cfg["l"], cfg["batch"], cfg["eps"]
    N = 4 * l - 1
    nthreads = max(1, (os.cpu_count() or 1) // max(1, world))
    t0 = time.perf_counter()
    sh = bb.ShardedSHT.create(l, eps=eps, device=local, threads=nthreads)
    t_build = time.perf_counter() - t0
    lay = sh.layout
    beta_np = sht_oracle.random_coefficients(l, B, seed=1000, decaying_member=cfg.get("decaying"))
    mine = np.zeros_like(beta_np)
    from paper_0910_5435_b200.sharded import coefficient_slices
    for a, b in coefficient_slices(l, *lay.my_orders):
        mine[:, a:b] = beta_np[:, a:b]
    beta = torch.from_numpy(mine).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        slab = sh.synthesize(beta)
        back = sh.analyze(slab)
    torch.cuda.synchronize()
    rt = float((torch.linalg.vector_norm(back - beta) / torch.linalg.vector_norm(beta)).item())
    rt = allreduce_max(rt, world)
    if not rt <= 1e-9:
        raise SystemExit(f"bench: the sharded pipeline does not round-trip (rel l2 {rt:.3e}); refusing to report")
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    sampler = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    sampler.start()
    for k in range(K):
        flush.fill_(k & 0xFF)
        ev[k][0].record()
        slab = sh.synthesize(beta)
        back = sh.analyze(slab)
        ev[k][1].record()
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    t_step = allreduce_max(sum(e[0].elapsed_time(e[1]) for e in ev) / K, world)
    if rank == 0:
        line = {
            "metric": METRIC, "value": B / (t_step * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_block(args, cfg, 1), parallelism=f"orders sharded over {world} ranks, "
                           "NCCL all-to-all m<->theta transpose", global_batch=B),
            "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": None, "clocks": clocks,
            "mode": "sharded", "plan_build_s": t_build, "round_trip_rel_l2": rt,
        }
        print(json.dumps(line), flush=True)
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
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", choices=["replicas", "sharded"], default="replicas",
                    help="replicas: each GPU transforms its own batch (default, weak scaling); "
                         "sharded: the orders of one batch are split over the GPUs (strong scaling)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.mode == "sharded":
        run_sharded(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
