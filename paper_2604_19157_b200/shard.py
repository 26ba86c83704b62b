"""Multi-GPU partitioning of the hot path: one process per GPU,
no collective on the data path.

Sequences are independent and so are kv heads (a q head reads only
its own kv head, layout.py:65-69), so each rank owns a contiguous block of
sequences (batch sharding, BASELINE configs C3/C4) or of kv heads with their
q heads (C5, long single requests).  torch.distributed is used only for the
barrier / max-over-ranks timing and to gather outputs for verification after
timing; the helpers take any backend (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from typing import Optional

import torch

from .errors import ShapeError
from .layout import HeadLayout


def block_range(n: int, world: int, rank: int) -> range:
    """Contiguous block of [0, n) for `rank`: sizes differ by at most one, the
    first n % world ranks take the larger blocks."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ShapeError(f"bad partition n={n} world={world} rank={rank}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def shard_sequences(seqs, world: int, rank: int) -> list:
    """The sequences this rank serves (batch sharding)."""
    seqs = list(seqs)
    r = block_range(len(seqs), world, rank)
    return seqs[r.start:r.stop]


def shard_heads(layout: HeadLayout, world: int, rank: int) -> tuple[HeadLayout, range, range]:
    """kv-head sharding of one request: (this rank's layout, its kv heads, its q heads).
    num_kv_heads must be a multiple of world so every rank runs the same kernel shape."""
    if layout.num_kv_heads % world:
        raise ShapeError(f"{layout.num_kv_heads} kv heads do not split over {world} ranks")
    kv = block_range(layout.num_kv_heads, world, rank)
    g = layout.group_size
    local = HeadLayout(num_q_heads=len(kv) * g, num_kv_heads=len(kv), head_dim=layout.head_dim,
                       rot_order=layout.rot_order, page_tokens=layout.page_tokens)
    return local, kv, range(kv.start * g, kv.stop * g)


def max_over_ranks(value: float, device: Optional[torch.device] = None) -> float:
    """Max of a per-rank scalar (the bench's timing rule); identity without a process group."""
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor, counts: list[int]) -> torch.Tensor:
    """Concatenate every rank's leading-dim block (block sizes `counts`, as from
    block_range) in rank order; all_gather needs equal shapes, so blocks are padded."""
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return local
    world = torch.distributed.get_world_size()
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    torch.distributed.all_gather(parts, pad)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
