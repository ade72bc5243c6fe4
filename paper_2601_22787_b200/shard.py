"""Multi-GPU sharding of the decode hot path.

The work shards by transformer block: blocks are independent (own table, own chunks), so
ranks need no data-path collective.  Only the timing uses collectives (barrier + MAX).
"""
from __future__ import annotations


def layer_ids(rank: int, world: int, blocks: int, scaling: str = "weak") -> list[int]:
    """Block (layer) ids decoded by ``rank``.

    weak:   every rank decodes its own ``blocks``-block layer set (distinct ids
            rank*blocks .. rank*blocks+blocks-1) — per-GPU work fixed as N grows.
    strong: one ``blocks``-block layer set split round-robin over the ranks."""
    if world < 1 or not (0 <= rank < world) or blocks < 1:
        raise ValueError("bad rank/world/blocks")
    if scaling == "weak":
        return [rank * blocks + i for i in range(blocks)]
    if scaling == "strong":
        return [i for i in range(blocks) if i % world == rank]
    raise ValueError(scaling)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """MAX of a per-rank scalar (elapsed ms) over the process group (identity when single)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_gbs(bytes_per_rank: float, world: int, steps: int, max_ms: float) -> float:
    """Whole-job throughput: all ranks' algorithmic bytes over the slowest rank's time."""
    return bytes_per_rank * world * steps / (max_ms / 1e3) / 1e9
