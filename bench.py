#!/usr/bin/env python3
"""Benchmark of the FFS hot path (BASELINE.json metric: FFS samples/sec and effective FP64
GFLOP/s at 1 B200; % of roofline).

One "step" = one ffs_sample call over the whole workload (permutation draw, candidate weights,
inverse-CDF draws, panel/factor updates, positions out for all M samples) with inputs resident in
HBM. Default workload: BASELINE.json configs[1] (1D double well, L=256, N=32, M=65536, fp64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config dw] [--impl reference]

N>1: launched under torchrun (one process per GPU); every rank samples its own M samples (own
uniform stream, "scaling": "weak"), no collective on the data path; the timed region is bracketed
by a barrier + synchronize and the max over ranks is reported.
`--impl reference` times the CPU oracle (oracle/, the paper's algorithm in C) on a bounded
sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2109_07358_b200 import inputs  # noqa: E402

METRIC = "FFS samples/sec and effective FP64 GFLOP/s vs (L,N) at 1 B200; % of roofline"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP64 FMA pipe: 148 SMs x 64 FMA/clk x 2 flop x 1.965 GHz (measured: DMMA 36.9,
# DFMA 34.1, cuBLAS DGEMM 35.5 TFLOP/s — profiles/fp64_peaks_r01.json)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel per launch, from one
# `ncu --set full` capture of this bench command (profiles/r01_ncu_summary.md)
TRAFFIC_BYTES = {"dw": 25294336}


def paper_flops(cfg_L, Np, cplx):
    """Algorithmic flops per sample, PAPER.md:81/83 (L N'^2 + N'^3; x4 for complex)."""
    return (4 if cplx else 1) * (cfg_L * Np * Np + Np ** 3)


def weight_flops(cfg_L, Np, cplx):
    """Candidate-weight flops per sample: sum_k 2 L k."""
    return (4 if cplx else 1) * cfg_L * Np * (Np + 1)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[2 + j].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(name, marginal, rank):
    cfg = inputs.CONFIGS[name]
    U = inputs.build_u(cfg)
    if marginal:
        M, Np = cfg.marginal_M, cfg.marginal_Np
        uni = inputs.uniforms(M, Np, cfg.uniform_seed + 100 + 7919 * rank)
    else:
        M, Np = cfg.M, cfg.N
        uni = inputs.uniforms(M, Np, cfg.uniform_seed + 7919 * rank)
    return cfg, U, uni, M, Np


def cpu_oracle_rate(U, uni, Np, budget_s=15.0, max_samples=None):
    """Oracle samples/s on a bounded prefix of the workload (host cores, OpenMP)."""
    from oracle import ref
    ref.lib()
    L = U.shape[0]
    work = (4 if np.iscomplexobj(U) else 1) * (L * Np * Np + Np ** 3)
    # one sample per host thread first, except where one sample is already ~10+ s of CPU work
    # (C5 full: 1.8e10 flop per sample; 16 concurrent samples took 217 s, memory-bound)
    n = 1 if work > 8e9 else max(1, ref.num_threads())
    t_used = 0.0
    while True:
        n = min(n, uni.shape[0] if max_samples is None else min(uni.shape[0], max_samples))
        t0 = time.perf_counter()
        ref.sample(U, uni[:n], Np=Np)
        t = time.perf_counter() - t0
        if t > budget_s / 4 or n >= uni.shape[0] or (max_samples and n >= max_samples):
            t_used = t
            break
        n = int(n * max(2.0, min(16.0, (budget_s / 4) / max(t, 1e-3))))
    return n / t_used, n, t_used, min(n, ref.num_threads())  # threads actually used (OpenMP over samples)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg, U, uni, M, Np = workload(args.config, args.marginal, 0)
    cplx = np.iscomplexobj(U)
    rates = []
    n_used = 0
    for step in range(args.warmup + args.steps):
        rate, n, t, cores = cpu_oracle_rate(U, uni, Np, budget_s=min(20.0, 60.0 / max(1, args.steps)))
        if step >= args.warmup:
            rates.append(rate)
            n_used = n
    v = statistics.median(rates)
    ms = M / v * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128" if cplx else "f64", "data": "synthetic",
        "config": {"workload": cfg.name + (":marginal" if args.marginal else ""), "L": cfg.L, "N": cfg.N,
                   "Nprime": Np, "M": M, "per_step_sample": f"first {n_used} of {M} samples"},
        "effective_gflops": v * paper_flops(cfg.L, Np, cplx) / 1e9,
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {n_used} samples of the workload per step, OpenMP over samples"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2109_07358_b200 import ffs

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg, U, uni, M, Np = workload(args.config, args.marginal, rank)
    cplx = np.iscomplexobj(U)
    Ud = torch.from_numpy(np.ascontiguousarray(U)).to(dev)
    ud = torch.from_numpy(uni).to(dev)
    pos = torch.empty((M, Np), dtype=torch.int32, device=dev)
    flg = torch.empty(M, dtype=torch.int32, device=dev)
    ws = ffs.Workspace(dev)
    stream = torch.cuda.current_stream(dev)
    # L2 flush buffer (> 126 MB L2): the workload's inputs are smaller than L2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        ffs.ffs_sample_marginal(Ud, ud, Np, positions=pos, flags=flg, workspace=ws, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    ffs.ffs_profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local)
    clk.start()
    total_ms = 0.0
    kern_ms = []
    launches = 0
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
        kern_ms.append(ffs.ffs_last_kernel_ms())
        launches += ffs.ffs_last_launch_count()
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ffs.ffs_profile_enable(False)
    ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    flags_bad = int((flg != 0).sum().item())

    # ---- end-to-end through the host-buffer C-ABI call (pinned host buffers, copies timed)
    hU = torch.from_numpy(np.ascontiguousarray(U)).pin_memory()
    hu = torch.from_numpy(uni).pin_memory()
    hp = torch.empty((M, Np), dtype=torch.int32).pin_memory()
    hf = torch.empty(M, dtype=torch.int32).pin_memory()
    hws = ffs.Workspace(dev)
    for _ in range(max(1, args.warmup // 2)):
        ffs.ffs_sample_host(hU, hu, Np, positions=hp, flags=hf, workspace=hws, stream=stream, device=dev)
    e2e_ms = []
    for _ in range(args.steps):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        ffs.ffs_sample_host(hU, hu, Np, positions=hp, flags=hf, workspace=hws, stream=stream, device=dev)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e = statistics.median(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())
    assert (hp.to(dev) == pos).all().item(), "host path and device path disagree"

    if rank == 0:
        units = M * world
        value = units / (ms * 1e-3)
        fl = paper_flops(cfg.L, Np, cplx)
        kms = statistics.median([k for k in kern_ms if k > 0]) if any(k > 0 for k in kern_ms) else ms
        achieved = M * fl / (kms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128" if cplx else "f64", "data": "synthetic",
            "config": {"workload": cfg.name + (":marginal" if args.marginal else ""), "L": cfg.L, "N": cfg.N,
                       "Nprime": Np, "M_per_gpu": M, "l2": "flushed (256 MB write) before every timed step",
                       "U_sha256": inputs.u_sha256(U)[:16]},
            "effective_gflops": value * fl / 1e9,
            "weight_gflops": value * weight_flops(cfg.L, Np, cplx) / 1e9,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                         "kernel": ffs_path_kernel(cfg, Np, cplx),
                         "kernel_ms": kms, "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"},
            "gpu_launches": launches,
            "sample_flags_nonzero": flags_bad,
            "clocks": clocks,
            "e2e": {"value": units / (e2e * 1e-3), "unit": "samples/s",
                    "h2d_bytes_per_step": int(hU.numel() * hU.element_size() + hu.numel() * 8),
                    "d2h_bytes_per_step": int(hp.numel() * 4 + hf.numel() * 4)},
        }
        if args.traffic is not None:
            line["roofline"]["traffic"] = args.traffic
        elif not args.marginal and cfg.name in TRAFFIC_BYTES:
            line["roofline"]["traffic"] = TRAFFIC_BYTES[cfg.name]
        if not args.no_cpu and world == 1:
            rate, n, t, cores = cpu_oracle_rate(U, uni, Np, budget_s=args.cpu_budget)
            line["cpu_baseline"] = {"value": rate, "unit": "samples/s", "cores": cores, "kind": "oracle",
                                    "sample": f"first {n} of {M} samples ({t:.1f} s), OpenMP over samples"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def ffs_uses_warp(cfg, Np, cplx):
    return (not cplx) and cfg.L <= 256 and Np <= 48


def ffs_path_kernel(cfg, Np, cplx):
    """Name of the timed kernel (sequence) of the path libffs dispatches to (ffs_abi.cu launch())."""
    if ffs_uses_warp(cfg, Np, cplx):
        return "ffs_seg_kernel"
    if cfg.L >= 2048:
        if Np < cfg.N and cfg.N >= 256 and cfg.N % 2 == 0:
            return "step path (marginal): ffs_cluster_kernel<STEP> (gathered contraction) + ffs_dense_gj_kernel per block"
        if Np == cfg.N and cfg.N >= 256 and cfg.N % 2 == 0:
            return ("dense path (hybrid): ffs_cluster_kernel<STEP> (+ ffs_ozaki_gemm_kernel for k0 >= theta N') "
                    "+ ffs_dense_gj_kernel per block")
        return "ffs_cluster_kernel"
    return "ffs_sample_kernel"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="dw", choices=sorted(inputs.CONFIGS))
    ap.add_argument("--marginal", action="store_true", help="the config's marginal (N'<N) workload")
    ap.add_argument("--impl", default="ffs", choices=["ffs", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the dominant kernel from an ncu --set full capture")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
