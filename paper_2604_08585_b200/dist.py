"""Request sharding across GPUs.

Requests are independent (fusion.py:211-216: the engine is shared read-only),
so there is no data-path collective: rank r serves a contiguous block of the
request list on its own GPU, and one gather at the end brings the per-request
results (first-token logits, selected positions, device times) to rank 0.
One process per GPU; backend "nccl" on the B200 box, "gloo" in CPU tests.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from torchrun's environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(n_items: int, world: int, rank: int) -> range:
    """Contiguous block of the item list owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, rem = divmod(n_items, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def gather_rows(local: torch.Tensor, n_total: int, world: int, rank: int,
                group=None) -> torch.Tensor | None:
    """Gather per-request rows `local` [n_local, ...] from every rank into
    [n_total, ...] on rank 0 (others get None). Blocks are padded to the
    largest block so one all_gather_into_tensor (NCCL or gloo) suffices."""
    if world == 1:
        return local
    per = -(-n_total // world)
    pad = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    out = torch.empty((per * world,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "gloo":   # CPU tests / single-GPU multi-rank testing
        pad_h = pad.cpu()
        parts = [torch.empty_like(pad_h) for _ in range(world)]
        dist.all_gather(parts, pad_h, group=group)
        out = torch.cat(parts).to(local.device)
    else:
        dist.all_gather_into_tensor(out, pad, group=group)
    if rank != 0:
        return None
    rows = [out[r * per: r * per + len(shard(n_total, world, r))] for r in range(world)]
    return torch.cat(rows)


def max_over_ranks(value: float, device, group=None) -> float:
    """Max of a scalar over ranks (multi-GPU times are max-over-ranks)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    on_gloo = dist.get_backend(group) == "gloo"
    t = torch.tensor([value], dtype=torch.float64, device="cpu" if on_gloo else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
