"""Sample sharding across ranks (one process per GPU). Samples are independent
(PAPER.md:82), so a rank owns a contiguous range of sample rows — of the uniforms and of the
positions — and no collective is needed on the data path. `gather_positions` is the optional
post-processing all-gather for a caller that wants every rank's positions."""
from __future__ import annotations


def shard_range(M: int, rank: int, world: int):
    """Contiguous [lo, hi) of the M samples owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world) or M < 0:
        raise ValueError((M, rank, world))
    base, extra = divmod(M, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_positions(local, M: int, group=None):
    """All-gather the per-rank position blocks into the full [M][N'] array (torch.distributed)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_range(M, r, world) for r in range(world)]
    width = local.shape[1]
    mx = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros((mx, width), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[: hi - lo] for o, (lo, hi) in zip(out, sizes)], dim=0)
