#!/usr/bin/env python3
"""Benchmark of the FFS hot path (BASELINE.json metric: FFS samples/sec and effective FP64
GFLOP/s vs (L,N) at 1 B200; % of roofline).

One "step" = one ffs_sample call over the whole workload (permutation draw, candidate weights,
inverse-CDF draws, panel/factor updates, positions out for all M samples) with inputs resident in
HBM. Default workload: the largest single-GPU configuration of BASELINE.json, configs[4] (the
DPP-shaped projection DPP, L=16384, N=1024, M=1024, fp64). The same JSON line carries a `sweep`
with every BASELINE.json workload (C1, C2, C3, C3 marginal, C4, C5, C5 marginal), each timed the
same way (device time, kernel time, roofline fraction, clocks, end-to-end through the host-buffer
C-ABI call, and the CPU oracle on a bounded sample).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config dpp] [--marginal] [--no-sweep]
  python bench.py --impl reference     # the CPU oracle (oracle/) as the reference arm

N>1: launched under torchrun (one process per GPU); every rank samples its own M samples (own
uniform stream, "scaling": "weak"), no collective on the data path; the timed region is bracketed
by a barrier + synchronize and the max over ranks is reported (the sweep runs at N=1 only).
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
# FP64 FMA pipe: 148 SMs x 64 FMA/clk x 2 flop x 1.965 GHz (measured on this pool:
# DMMA 36.9, DFMA 34.1, cuBLAS DGEMM 35.5 TFLOP/s, profiles/fp64_peaks_r01.json).
# MEASURED_PEAKS.json has no FP64 entry, so the derived peak is the denominator.
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# ncu-measured per-launch numbers of this round (tools/gpu_r2_ncu.sh): DRAM traffic of the
# dominant kernel and, for the dense path, the INT8 tensor-pipe activity of its GEMM
ROOFLINE_FILE = os.path.join(ROOT, "profiles", "roofline_r02.json")
SWEEP = [("tiny", False), ("dw", False), ("anderson", False), ("anderson", True), ("peierls", False),
         ("dpp", False), ("dpp", True)]
L2_NOTE = "flushed (256 MB write) before every timed GPU step"


def paper_flops(L, Np, cplx):
    """Algorithmic flops per sample, PAPER.md:81/83 (L N'^2 + N'^3; x4 for complex)."""
    return (4 if cplx else 1) * (L * Np * Np + Np ** 3)


def weight_flops(L, Np, cplx):
    """Candidate-weight flops per sample: sum_k 2 L k."""
    return (4 if cplx else 1) * L * Np * (Np + 1)


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


def workload(name, marginal, rank, world=1):
    cfg = inputs.CONFIGS[name]
    # multi-GPU: U is built once, on rank 0, and broadcast (broadcast_u); every rank
    # draws its own uniform stream
    U = inputs.build_u(cfg) if rank == 0 or world == 1 else None
    if marginal:
        M, Np = cfg.marginal_M, cfg.marginal_Np
        uni = inputs.uniforms(M, Np, cfg.uniform_seed + 100 + 7919 * rank)
    else:
        M, Np = cfg.M, cfg.N
        uni = inputs.uniforms(M, Np, cfg.uniform_seed + 7919 * rank)
    return cfg, U, uni, M, Np


def wl_name(name, marginal):
    return name + (":marginal" if marginal else "")


def config_of(cfg, Np, M):
    """The `config` object of both arms (identical keys and values)."""
    return {"workload": wl_name(cfg.name, Np < cfg.N), "L": cfg.L, "N": cfg.N, "Nprime": Np, "M": M,
            "l2": L2_NOTE}


def km_np_max(L):
    """Largest N' the tile-Gram path takes (ffs_abi.cu kmarg_eligible)."""
    return 24 if L <= 1024 else 32 if L < 2048 else 64 if L < 4096 else 96


def path_of(cfg, Np, cplx):
    """Kernel (sequence) libffs dispatches this shape to (ffs_abi.cu launch()) and its arithmetic."""
    if (not cplx) and cfg.L <= 256 and Np <= 48:
        return "ffs_seg_kernel (warp-segment owners)", "f64"
    dt = "c128" if cplx else "f64"
    if (not cplx) and Np <= km_np_max(cfg.L) and 64 * Np <= 3 * cfg.L and cfg.N <= 2048:
        return ("tile-Gram path: ffs_tile_gram_u_kernel (32 tile Gram matrices of U, once per call) + "
                "ffs_kmarg_kernel (warp per sample, tile totals as quadratic forms"
                + (", blocked)" if Np > 32 else ")")), dt
    if cfg.L >= 2048 and cfg.N >= 256 and cfg.N % 2 == 0:
        if Np < cfg.N:
            return ("block-step path (marginal): ffs_cluster_kernel<STEP> (gathered contraction, panel out) + "
                    "ffs_gram_kernel + ffs_gram_draw_kernel + ffs_dense_gj(2)_kernel per block, CUDA graph"), dt
        return ("block-step path (hybrid dense): per block ffs_ozaki_gemm2w_kernel (P = U Y; gathered contraction in "
                "ffs_cluster_kernel<STEP> for k0 < theta N'), ffs_gram_kernel + ffs_gram_draw_kernel (draws on tile "
                "Gram matrices, warp per sample), ffs_dense_gj_kernel / ffs_dense_gj2_kernel; CUDA graph"), \
            dt + " (dense GEMM: Ozaki FP64 emulation, int8 x 8 slices on tcgen05; fp64-level, <= 1.3e-15 normwise)"
    if cfg.L >= 2048:
        return "ffs_cluster_kernel", dt
    return "ffs_sample_kernel (CTA owners)", dt


def path_note(cfg, Np, cplx):
    """What `frac` means where the path executes fewer flops than the paper's count."""
    if (not cplx) and not (cfg.L <= 256 and Np <= 48) and Np <= km_np_max(cfg.L) and 64 * Np <= 3 * cfg.L and cfg.N <= 2048:
        return ("tile-Gram path: tile totals come from the tile Gram matrices of U, so the executed flops per sample "
                "(~G N'^3/6 + N'^2 L/(2G), G = 16 or 32 tiles) are below the paper's L N'^2 + N'^3 that `achieved` "
                "counts; frac is a throughput ratio against the FP64 peak, not a pipe utilisation")
    return None


def load_roofline_file():
    try:
        with open(ROOFLINE_FILE) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_oracle_rate(U, uni, Np, budget_s=15.0):
    """Oracle samples/s on a bounded prefix of the workload (host cores, OpenMP over samples)."""
    from oracle import ref
    ref.lib()
    L = U.shape[0]
    work = (4 if np.iscomplexobj(U) else 1) * (L * Np * Np + Np ** 3)
    # one sample per host thread first, except where one sample is already ~10+ s of CPU work
    # (C5 full: 1.8e10 flop per sample; 16 concurrent samples took 217 s, memory-bound)
    n = 1 if work > 8e9 else max(1, ref.num_threads())
    while True:
        n = min(n, uni.shape[0])
        t0 = time.perf_counter()
        ref.sample(U, uni[:n], Np=Np)
        t = time.perf_counter() - t0
        if t > budget_s / 4 or n >= uni.shape[0]:
            break
        n = int(n * max(2.0, min(16.0, (budget_s / 4) / max(t, 1e-3))))
    return n / t, n, t, min(n, ref.num_threads())  # threads actually used (OpenMP over samples)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg, U, uni, M, Np = workload(args.config, args.marginal, 0)
    cplx = np.iscomplexobj(U)
    rates, n_used, cores = [], 0, 1
    for step in range(args.warmup + args.steps):
        rate, n, t, cores = cpu_oracle_rate(U, uni, Np, budget_s=min(20.0, 60.0 / max(1, args.steps)))
        if step >= args.warmup:
            rates.append(rate)
            n_used = n
    v = statistics.median(rates)
    _, dt = path_of(cfg, Np, cplx)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": M / v * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128" if cplx else "f64", "data": "synthetic",
        "config": config_of(cfg, Np, M),
        "effective_gflops": v * paper_flops(cfg.L, Np, cplx) / 1e9,
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {n_used} of {M} samples per step (extrapolated to M), OpenMP over samples"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def broadcast_u(U, cfg, dev, world):
    """U on this rank's device: rank 0's bytes, sent to the others with one broadcast (NCCL on the
    GPU box; any torch.distributed backend), outside every timed region."""
    import torch
    if world == 1:
        return torch.from_numpy(np.ascontiguousarray(U)).to(dev)
    import torch.distributed as dist
    dt = torch.complex128 if cfg.dtype == inputs.C128 else torch.float64
    if U is not None:
        Ud = torch.from_numpy(np.ascontiguousarray(U)).to(dev)
    else:
        Ud = torch.empty((cfg.L, cfg.N), dtype=dt, device=dev)
    if dt == torch.complex128:
        dist.broadcast(torch.view_as_real(Ud), src=0)
    else:
        dist.broadcast(Ud, src=0)
    return Ud


def measure_gpu(name, marginal, steps, warmup, rank, world, dev, with_e2e=True):
    """Device-time samples/s of one workload (inputs resident, L2 flushed before every step),
    the libffs kernel time, clocks during the timed region, and the host-buffer e2e rate."""
    import torch
    import torch.distributed as dist
    from paper_2109_07358_b200 import ffs

    cfg, U, uni, M, Np = workload(name, marginal, rank, world)
    Ud = broadcast_u(U, cfg, dev, world)
    if U is None:
        U = Ud.cpu().numpy()  # the host copy for the e2e leg (the bytes rank 0 built)
    cplx = np.iscomplexobj(U)
    ud = torch.from_numpy(uni).to(dev)
    pos = torch.empty((M, Np), dtype=torch.int32, device=dev)
    flg = torch.empty(M, dtype=torch.int32, device=dev)
    ws = ffs.Workspace(dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        ffs.ffs_sample_marginal(Ud, ud, Np, positions=pos, flags=flg, workspace=ws, stream=stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    ffs.ffs_profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(dev.index or 0)
    clk.start()
    total_ms, kern_ms, launches = 0.0, [], 0
    for _ in range(steps):
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
    ms = total_ms / steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    flags_bad = int((flg != 0).sum().item())
    kms = statistics.median([k for k in kern_ms if k > 0]) if any(k > 0 for k in kern_ms) else ms
    fl = paper_flops(cfg.L, Np, cplx)
    achieved = M * fl / (kms * 1e-3) / 1e12
    out = {"cfg": cfg, "U": U, "uni": uni, "M": M, "Np": Np, "cplx": cplx, "ms": ms, "kernel_ms": kms,
           "achieved": achieved, "frac": achieved / FP64_PEAK_TFLOPS, "clocks": clocks,
           "launches": launches, "flags_bad": flags_bad, "steps": steps}
    del flush
    if with_e2e:
        # end to end through the host-buffer C-ABI call (pinned host buffers, copies timed)
        hU = torch.from_numpy(np.ascontiguousarray(U)).pin_memory()
        hu = torch.from_numpy(uni).pin_memory()
        hp = torch.empty((M, Np), dtype=torch.int32).pin_memory()
        hf = torch.empty(M, dtype=torch.int32).pin_memory()
        hws = ffs.Workspace(dev)
        ffs.ffs_sample_host(hU, hu, Np, positions=hp, flags=hf, workspace=hws, stream=stream, device=dev)
        e2e_ms = []
        for _ in range(steps):
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
        out["e2e"] = {"value": M * world / (e2e * 1e-3), "unit": "samples/s",
                      "h2d_bytes_per_step": int(hU.numel() * hU.element_size() + hu.numel() * 8),
                      "d2h_bytes_per_step": int(hp.numel() * 4 + hf.numel() * 4)}
        del hws
    del ws, Ud, ud
    torch.cuda.empty_cache()
    return out


def sweep_entry(r, cpu_budget, no_cpu):
    cfg, M, Np, cplx = r["cfg"], r["M"], r["Np"], r["cplx"]
    kern, dt = path_of(cfg, Np, cplx)
    e = {"config": config_of(cfg, Np, M), "dtype": dt, "value": M / (r["ms"] * 1e-3), "unit": "samples/s",
         "ms_per_step": r["ms"], "steps": r["steps"], "kernel": kern, "kernel_ms": r["kernel_ms"],
         "effective_gflops": M * paper_flops(cfg.L, Np, cplx) / (r["ms"] * 1e-3) / 1e9,
         "frac": r["frac"], "clocks": r["clocks"], "e2e": r.get("e2e"), "gpu_launches": r["launches"],
         "sample_flags_nonzero": r["flags_bad"]}
    if path_note(cfg, Np, cplx):
        e["note"] = path_note(cfg, Np, cplx)
    if not no_cpu:
        rate, n, t, cores = cpu_oracle_rate(r["U"], r["uni"], Np, budget_s=cpu_budget)
        e["cpu_baseline"] = {"value": rate, "unit": "samples/s", "cores": cores, "kind": "oracle",
                             "sample": f"first {n} of {M} samples ({t:.1f} s), OpenMP over samples"}
    return e


def measure_extensions(dev, steps, no_cpu, cpu_budget):
    """The §8(f) rows beyond the BASELINE workloads, each timed like a sweep entry (device time
    with inputs resident, L2 flushed, kernel events, clocks, e2e where a host path exists):
    the L-ensemble front end (`lens`), the Supp S7 Metropolis variant (`metro`), the
    Gutzwiller reweighting of C2 spinful samples (`gutzwiller`, HBM-bound), small-N' marginals at
    L = 65536 (`large_L`, `large_L_complex`) and the modified-HKPV comparator."""
    import torch
    from paper_2109_07358_b200 import ffs

    out = {}
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn, K):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        ffs.ffs_profile_enable(True)
        clk = ClockSampler(dev.index or 0)
        clk.start()
        tot, kms = 0.0, []
        for _ in range(K):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
            kms.append(ffs.ffs_last_kernel_ms())
        clocks = clk.stop()
        ffs.ffs_profile_enable(False)
        return tot / K, statistics.median(kms), clocks, ffs.ffs_last_launch_count()

    # L-ensemble
    cfg = inputs.LENS
    V, lam = inputs.build_lensemble(cfg)
    uni = inputs.lens_uniforms(cfg.M, cfg.D, cfg.uniform_seed)
    Vd, ld, ud = (torch.from_numpy(a).to(dev) for a in (V, lam, uni))
    ws = ffs.Workspace(dev)
    res = {}

    def lens_step():
        res["out"] = ffs.ffs_sample_lensemble(Vd, ld, ud, workspace=ws, stream=stream)

    ms, kms, clocks, nl = timed(lens_step, steps)
    nmean = float(res["out"][1].double().mean().item())
    fl = cfg.L * nmean ** 2 + nmean ** 3  # PAPER.md:81 at the sample's own N_i (mean)
    out["lens"] = {"config": {"workload": "lens", "L": cfg.L, "K": cfg.D, "mean_N": nmean, "M": cfg.M,
                              "l2": L2_NOTE},
                   "dtype": "f64", "value": cfg.M / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms,
                   "kernel": "ffs_lens_prep_kernel + ffs_sample_kernel (ragged mode, CTA owners)",
                   "kernel_ms": kms, "effective_gflops": cfg.M * fl / (ms * 1e-3) / 1e9,
                   "frac": cfg.M * fl / (kms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, "clocks": clocks, "gpu_launches": nl}
    if not no_cpu:
        from oracle import ref
        n = 2048
        t0 = time.perf_counter()
        ref.sample_lensemble(V, lam, uni[:n])
        t = time.perf_counter() - t0
        out["lens"]["cpu_baseline"] = {"value": n / t, "unit": "samples/s", "cores": min(n, ref.num_threads()),
                                       "kind": "oracle", "sample": f"first {n} of {cfg.M} samples ({t:.1f} s)"}
    del Vd, ld, ud, ws

    # Supp S7 Metropolis variant, continuous-model stand-in (L = 2^20 grid)
    mc = inputs.METRO
    U = inputs.build_box_orbitals(mc.L, mc.N)
    uni = inputs.metro_uniforms(mc.M, mc.N, mc.Mc, mc.uniform_seed)
    Ud, ud = torch.from_numpy(U).to(dev), torch.from_numpy(uni).to(dev)
    ws = ffs.Workspace(dev)

    def metro_step():
        ffs.ffs_sample_metropolis(Ud, ud, mc.N, mc.Mc, workspace=ws, stream=stream)

    ms, kms, clocks, nl = timed(metro_step, steps)
    N = mc.N
    fl = N ** 3 / 3 + 2 * mc.Mc * N * (N + 1) / 2      # GJ rank-1 updates + Mc weights per step
    byts = 8 * mc.Mc * N * (N + 1) / 2 + 16 * N * (1 + 2 * mc.Mc)  # gathered U entries + uniforms
    out["metro"] = {"config": {"workload": "metro", "L": mc.L, "N": N, "Nprime": N, "Mcond": mc.Mc, "M": mc.M,
                               "l2": L2_NOTE},
                    "dtype": "f64", "value": mc.M / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms,
                    "kernel": "ffs_permute_kernel + ffs_metro_kernel (warp per sample)", "kernel_ms": kms,
                    "roofline": {"bound": "hbm", "achieved": mc.M * byts / (kms * 1e-3) / 1e9,
                                 "peak": measured_hbm(), "unit": "GB/s",
                                 "frac": mc.M * byts / (kms * 1e-3) / 1e9 / measured_hbm(),
                                 "bytes_def": "algorithmic: the gathered U entries of every chain state "
                                              "(8 (k+1) B per state) + the chain uniforms, per sample"},
                    "effective_gflops": mc.M * fl / (ms * 1e-3) / 1e9, "clocks": clocks, "gpu_launches": nl}
    if not no_cpu:
        from oracle import ref
        n = 256
        t0 = time.perf_counter()
        ref.sample_metropolis(U, uni[:n], N, mc.Mc)
        t = time.perf_counter() - t0
        out["metro"]["cpu_baseline"] = {"value": n / t, "unit": "samples/s", "cores": min(n, ref.num_threads()),
                                        "kind": "oracle", "sample": f"first {n} of {mc.M} samples ({t:.1f} s)"}
    del Ud, ud, ws

    # Gutzwiller reweighting (Supp S5) of C2 spinful samples: an HBM-bound reduction
    cfg, U, uni, M, Np = workload("dw", False, 0)
    pos = ffs.ffs_sample(torch.from_numpy(U).to(dev), torch.from_numpy(uni).to(dev))
    ws = ffs.Workspace(dev)

    def gw_step():
        ffs.ffs_gutzwiller_reweight(pos, cfg.L, 1.0, workspace=ws, stream=stream)

    ms, kms, clocks, nl = timed(gw_step, steps)
    byts = M * Np * 4
    out["gutzwiller"] = {"config": {"workload": "gutzwiller(dw)", "L": cfg.L, "Nprime": Np, "spinful_samples": M // 2,
                                    "V": 1.0, "l2": L2_NOTE},
                         "value": (M // 2) / (ms * 1e-3), "unit": "spinful samples/s", "ms_per_step": ms,
                         "kernel": "ffs_gutzwiller_kernel + ffs_reweight_finalize_kernel", "kernel_ms": kms,
                         "roofline": {"bound": "hbm", "achieved": byts / (kms * 1e-3) / 1e9, "peak": measured_hbm(),
                                      "unit": "GB/s", "frac": byts / (kms * 1e-3) / 1e9 / measured_hbm(),
                                      "bytes_def": "positions read once: 4 N' B per sample"},
                         "clocks": clocks, "gpu_launches": nl}
    # L beyond the panel kernels' limits (16384 real / 8192 complex): small-N' marginals on the tile-Gram path
    for cx in (False, True):
        L, N, Np, M = 65536, 64, 16, 4096
        U = inputs.random_orthonormal(L, N, 5000 + N, complex_=cx)
        uni = inputs.uniforms(M, Np, 5100 + int(cx))
        Ud, ud = torch.from_numpy(U).to(dev), torch.from_numpy(uni).to(dev)
        ws = ffs.Workspace(dev)
        ms, kms, clocks, nl = timed(lambda: ffs.ffs_sample_marginal(Ud, ud, Np, workspace=ws, stream=stream), steps)
        fl = paper_flops(L, Np, cx)
        key = "large_L_complex" if cx else "large_L"
        out[key] = {"config": {"workload": key, "L": L, "N": N, "Nprime": Np, "M": M, "l2": L2_NOTE},
                    "dtype": "c128" if cx else "f64", "value": M / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms,
                    "kernel": "ffs_tile_gram_u%s_kernel + ffs_kmarg%s_kernel (chunked row scan)" % (("c", "c") if cx else ("", "")),
                    "kernel_ms": kms, "effective_gflops": M * fl / (ms * 1e-3) / 1e9,
                    "frac": M * fl / (kms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                    "note": "throughput ratio against the paper's flop count (the tile-Gram path executes fewer flops)",
                    "clocks": clocks, "gpu_launches": nl}
        if not no_cpu:
            from oracle import ref
            n = 64
            t0 = time.perf_counter()
            ref.sample(U, uni[:n], Np=Np)
            t = time.perf_counter() - t0
            out[key]["cpu_baseline"] = {"value": n / t, "unit": "samples/s", "cores": min(n, ref.num_threads()),
                                        "kind": "oracle", "sample": f"first {n} of {M} samples ({t:.1f} s)"}
        del Ud, ud, ws
    # the paper's comparator on the same GPU: modified HKPV (2 L N^2) vs FFS (L N^2 + N^3),
    # PAPER.md:81 "nearly the twice" / Fig. 3B (L = 1024 random U, N sweep); same uniforms layout
    hk = {}
    cases = [("dw", None), ("anderson", None), ("dpp", None)] + [("fig3b", n) for n in (16, 32, 64, 128)]
    for name, n in cases:
        if name == "fig3b":
            L, N, M = 1024, n, 16384
            U = inputs.random_orthonormal(L, N, 3000 + N)
        else:
            cfg = inputs.CONFIGS[name]
            L, N, M = cfg.L, cfg.N, cfg.M
            U = inputs.build_u(cfg)
        uni = inputs.uniforms(M, N, 4000 + N)
        Ud = torch.from_numpy(U).to(dev)
        ud = torch.from_numpy(uni).to(dev)
        us = torch.from_numpy(np.ascontiguousarray(uni[:, N:])).to(dev)
        ws1, ws2 = ffs.Workspace(dev), ffs.Workspace(dev)
        K = 2 if name == "dpp" else max(3, min(steps, 5))
        ms_f, _, clk_f, _ = timed(lambda: ffs.ffs_sample(Ud, ud, workspace=ws1, stream=stream), K)
        ms_h, _, clk_h, nl = timed(lambda: ffs.ffs_sample_hkpv(Ud, us, workspace=ws2, stream=stream), K)
        key = f"{name}_N{N}" if name == "fig3b" else name
        hk[key] = {"L": L, "N": N, "M": M, "ffs_ms": ms_f, "hkpv_ms": ms_h, "time_ratio_hkpv_over_ffs": ms_h / ms_f,
                   "flop_ratio_paper": 2 * L * N ** 2 / (L * N ** 2 + N ** 3),
                   "hkpv_samples_per_s": M / (ms_h * 1e-3), "ffs_samples_per_s": M / (ms_f * 1e-3),
                   "clocks": clk_h, "hkpv_gpu_launches": nl}
        del Ud, ud, us, ws1, ws2
        torch.cuda.empty_cache()
    out["hkpv_comparator"] = hk
    del flush
    return out


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6547.5  # MEASURED_PEAKS.json value of round 1 (same pool)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    head = measure_gpu(args.config, args.marginal, args.steps, args.warmup, rank, world, dev)
    sweep = None
    if world == 1 and not args.no_sweep and rank == 0:
        sweep = {}
        for name, marg in SWEEP:
            key = wl_name(name, marg)
            if name == args.config and marg == args.marginal:
                r = head
            else:
                r = measure_gpu(name, marg, max(3, min(args.steps, 10)), 3, rank, world, dev)
            sweep[key] = sweep_entry(r, args.sweep_cpu_budget, args.no_cpu)
            sys.stderr.write(f"sweep {key}: {sweep[key]['value']:.4g} samples/s, frac {sweep[key]['frac']:.3f}\n")
    if rank == 0:
        cfg, M, Np, cplx = head["cfg"], head["M"], head["Np"], head["cplx"]
        units = M * world
        value = units / (head["ms"] * 1e-3)
        fl = paper_flops(cfg.L, Np, cplx)
        kern, dt = path_of(cfg, Np, cplx)
        rf = load_roofline_file().get(wl_name(cfg.name, Np < cfg.N), {})
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "config": config_of(cfg, Np, M),
            "inputs": {"U_sha256": inputs.u_sha256(head["U"])[:16], "uniforms": "numpy Philox, seed 1000+index"},
            "effective_gflops": value * fl / 1e9,
            "weight_gflops": value * weight_flops(cfg.L, Np, cplx) / 1e9,
            "roofline": {"bound": "alu", "achieved": head["achieved"], "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": head["frac"], "traffic": rf.get("traffic"),
                         "kernel": kern, "kernel_ms": head["kernel_ms"],
                         "achieved_def": "M x F_paper (L N'^2 + N'^3, x4 complex; PAPER.md:81/83) / kernel_ms "
                                         "(CUDA events on the launch stream around the sampling kernels)",
                         "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz "
                                        "(MEASURED_PEAKS.json has no FP64 entry)"},
            "gpu_launches": head["launches"],
            "sample_flags_nonzero": head["flags_bad"],
            "clocks": head["clocks"],
            "e2e": head["e2e"],
        }
        for k in ("traffic_source", "gemm"):
            if k in rf:
                line["roofline"][k] = rf[k]
        if path_note(cfg, Np, cplx):
            line["roofline"]["note"] = path_note(cfg, Np, cplx)
        if world == 1 and not args.no_cpu:
            if sweep and wl_name(cfg.name, Np < cfg.N) in sweep and "cpu_baseline" in sweep[wl_name(cfg.name, Np < cfg.N)]:
                line["cpu_baseline"] = sweep[wl_name(cfg.name, Np < cfg.N)]["cpu_baseline"]
            else:
                rate, n, t, cores = cpu_oracle_rate(head["U"], head["uni"], Np, budget_s=args.cpu_budget)
                line["cpu_baseline"] = {"value": rate, "unit": "samples/s", "cores": cores, "kind": "oracle",
                                        "sample": f"first {n} of {M} samples ({t:.1f} s), OpenMP over samples"}
        if sweep is not None:
            line["sweep"] = sweep
        if world == 1 and not args.no_sweep:
            line["extensions"] = measure_extensions(dev, max(3, min(args.steps, 10)), args.no_cpu, args.sweep_cpu_budget)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="dpp", choices=sorted(inputs.CONFIGS))
    ap.add_argument("--marginal", action="store_true", help="the config's marginal (N'<N) workload")
    ap.add_argument("--impl", default="ffs", choices=["ffs", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-sweep", action="store_true", help="only the headline workload")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--sweep-cpu-budget", type=float, default=6.0, help="seconds of oracle work per sweep entry")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
