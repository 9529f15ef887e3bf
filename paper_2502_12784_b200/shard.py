"""(batch, head) sharding across ranks -- SURVEY 8(e).

The fused MHA path has no cross-(b,h) dependency, so a job of B*H heads is
split into contiguous slabs, one per rank: rank r of G owns flattened heads
[floor(r*BH/G), floor((r+1)*BH/G)).  In the [B, H, N, d] layout a slab is a
contiguous range of the flattened (b*h) axis, so a shard is a view -- no
re-layout and no collective on the data path.  NCCL (torch.distributed) is
used only *after* the hot path, to gather results to rank 0 for verification.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch


def shard_range(bh_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slab of the flattened (batch*head) axis owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return (rank * bh_total) // world, ((rank + 1) * bh_total) // world


def slab(t: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """View of heads [lo, hi) of a [B, H, ...] tensor as [hi-lo, ...] (contiguous)."""
    flat = t.reshape(t.shape[0] * t.shape[1], *t.shape[2:])
    return flat[lo:hi]


def gather_to_rank0(local: torch.Tensor, bh_total: int, group=None) -> torch.Tensor | None:
    """Gather every rank's [n_local, ...] slab into the full [bh_total, ...] tensor on
    rank 0 (None elsewhere).  Uneven slabs are padded to the largest one for the
    collective and trimmed afterwards."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(bh_total, world, r) for r in range(world)]
    max_n = max(hi - lo for lo, hi in sizes)
    # NCCL gathers device tensors in place; gloo (the CPU test path, and the shared-GPU
    # bench hook) gathers host copies
    dev = local.device
    via_host = dist.get_backend(group) == "gloo" and local.is_cuda
    src = local.cpu() if via_host else local
    pad = torch.zeros((max_n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    pad[: src.shape[0]] = src
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if rank != 0:
        return None
    out = torch.cat([b[: hi - lo] for b, (lo, hi) in zip(bufs, sizes)], dim=0)
    return out.to(dev) if via_host else out


def run_sharded(fn: Callable[..., Sequence[torch.Tensor]], inputs: Sequence[torch.Tensor], group=None):
    """Run `fn` on this rank's (b,h) slab of every [B, H, N, d] input (passed as
    [n_local, 1, N, d]) and gather each output to rank 0.  Returns the list of
    gathered [B*H, ...] outputs on rank 0, None on the other ranks."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, H = inputs[0].shape[:2]
    lo, hi = shard_range(B * H, world, rank)
    local_in = [slab(x, lo, hi).unsqueeze(1).contiguous() for x in inputs]
    outs = fn(*local_in)
    gathered = [gather_to_rank0(o.reshape(o.shape[0], *o.shape[2:]), B * H, group) for o in outs]
    return gathered if rank == 0 else None
