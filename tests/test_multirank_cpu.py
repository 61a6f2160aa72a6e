"""N>1 path on CPU: the sample sharding used by multi-GPU runs, with gloo at world size 2.
Sharded sampling (oracle stands in for the per-rank sampler: it is what the GPU path is compared
against) reassembled by the all-gather equals single-process sampling row for row, because every
sample consumes only its own uniform row."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_07358_b200 import inputs
from paper_2109_07358_b200.shard import gather_positions, shard_range


def test_shard_ranges_partition():
    for M in (0, 1, 7, 65536, 1001):
        for world in (1, 2, 3, 8):
            rs = [shard_range(M, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, U, uni, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ref
    M = uni.shape[0]
    lo, hi = shard_range(M, rank, world)
    local = torch.from_numpy(ref.sample(U, uni[lo:hi]))
    full = gather_positions(local, M)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process(tmp_path):
    from oracle import ref
    ref.build()
    U = inputs.random_orthonormal(40, 8, 3)
    uni = inputs.uniforms(333, 8, 9)
    out = str(tmp_path / "pos.npy")
    mp.spawn(_worker, args=(2, _free_port(), U, uni, out), nprocs=2, join=True)
    assert (np.load(out) == ref.sample(U, uni)).all()


def _bcast_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    cfg = inputs.CONFIGS["tiny"]
    cfg_c = inputs.Config("cplx_small", 12, 3, 8, 3, inputs.C128, 0, "none")
    U = inputs.build_u(cfg) if rank == 0 else None
    Ud = bench.broadcast_u(U, cfg, torch.device("cpu"), world)
    Uc = inputs.random_orthonormal(12, 3, 5, complex_=True) if rank == 0 else None
    Ucd = bench.broadcast_u(Uc, cfg_c, torch.device("cpu"), world)
    np.save(out_path + f".{rank}.npy", Ud.numpy())
    np.save(out_path + f".c{rank}.npy", Ucd.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_u_broadcast(tmp_path):
    """bench.py's multi-GPU input path: rank 0 builds U once and broadcasts it (real and complex);
    every rank ends with rank 0's bytes."""
    out = str(tmp_path / "u")
    mp.spawn(_bcast_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    U0 = inputs.build_u(inputs.CONFIGS["tiny"])
    Uc = inputs.random_orthonormal(12, 3, 5, complex_=True)
    for r in range(2):
        assert (np.load(out + f".{r}.npy") == U0).all()
        assert (np.load(out + f".c{r}.npy") == Uc).all()
