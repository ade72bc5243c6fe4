"""Multi-GPU sharding of the decode hot path.

The work shards by transformer block: blocks are independent (own table, own chunks), so
the decode itself needs no data-path collective (the bench: §8(e)'s contiguous 32/G split of
one layer set, barrier + MAX timing only).  Where a consumer needs blocks or tensors another rank holds, the exchange is
one all-gather: of compressed blocks (all_gather_blocks, decode locally) or of decoded row
shards (all_gather_rows).
"""
from __future__ import annotations


def layer_ids(rank: int, world: int, blocks: int, scaling: str = "strong") -> list[int]:
    """Block (layer) ids decoded by ``rank``.

    strong (default, SURVEY §8(e) for config 3): ONE ``blocks``-block layer set split into
            contiguous ranges, ``blocks``/world per rank (the first ``blocks`` % world ranks
            take one more) — 32/G blocks per GPU for Llama-3-8B; total work fixed as N grows.
    weak:   every rank decodes its own ``blocks``-block layer set (distinct ids
            rank*blocks .. rank*blocks+blocks-1) — per-GPU work fixed as N grows."""
    if world < 1 or not (0 <= rank < world) or blocks < 1:
        raise ValueError("bad rank/world/blocks")
    if scaling == "weak":
        return [rank * blocks + i for i in range(blocks)]
    if scaling == "strong":
        base, extra = divmod(blocks, world)
        lo = rank * base + min(rank, extra)
        return list(range(lo, lo + base + (1 if rank < extra else 0)))
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


# ---------------------------------------------------------------- exchange of compressed blocks
# when every rank needs every block (e.g. data-parallel inference with the
# compressed model sharded across GPUs, or "decode upcoming blocks on idle GPUs"), it
# is cheaper to all-gather the COMPRESSED blocks (≈ 2 bits/param) over NVLink and decode
# locally than to all-gather decoded bf16 weights (16 bits/param): ~8× fewer bytes on the
# link, and the local decode runs at HBM-class speed.  One collective per call: a byte
# tensor per rank holding its blocks back to back, padded to the largest rank's size.

def _blob_parts(b):
    """The device tensors of one Block in wire order (payload incl. decoder slack, offsets,
    table, scales), as uint8 views."""
    import torch
    keep = min(b.payload.numel(), b.payload_bytes + 256)          # EQ_PAYLOAD_SLACK
    return [b.payload[:keep], b.chunk_off.view(torch.uint8), b.freq.view(torch.uint8),
            b.scales.contiguous().view(torch.uint8)]


def pack_blocks(blocks):
    """(metadata list, one contiguous uint8 tensor) for a list of Blocks."""
    import torch
    meta, parts = [], []
    for b in blocks:
        ps = _blob_parts(b)
        meta.append({"sizes": [int(p.numel()) for p in ps], "payload_bytes": int(b.payload_bytes),
                     "shapes": [tuple(s) for s in b.shapes], "chunk_symbols": int(b.chunk_symbols),
                     "format": int(b.format), "codec": int(b.codec), "meta": dict(b.meta)})
        parts.extend(ps)
    flat = torch.cat(parts) if parts else torch.empty(0, dtype=torch.uint8)
    return meta, flat


def unpack_blocks(meta, flat):
    """Inverse of pack_blocks: Blocks whose tensors are views into (a copy of) ``flat``."""
    import torch
    from . import Block
    out, pos = [], 0
    for m in meta:
        sz = m["sizes"]
        seg = []
        for n in sz:
            seg.append(flat[pos:pos + n])
            pos += n
        payload = seg[0].clone()
        out.append(Block(payload, m["payload_bytes"], seg[1].clone().view(torch.int32), seg[2].clone().view(torch.int16),
                         seg[3].clone().view(torch.bfloat16), [tuple(s) for s in m["shapes"]], m["chunk_symbols"],
                         m["meta"], m["format"], m["codec"]))
    return out


def all_gather_blocks(blocks, dist, group=None):
    """Every rank's compressed blocks on every rank (rank-major order).  ``dist`` is
    torch.distributed (NCCL on GPUs; any backend works).  One all_gather of padded byte
    tensors plus one all_gather_object of the host metadata."""
    import torch
    world = dist.get_world_size(group)
    meta, flat = pack_blocks(blocks)
    metas = [None] * world
    dist.all_gather_object(metas, (meta, int(flat.numel())), group=group)
    n_max = max(n for _, n in metas)
    buf = torch.zeros(n_max, dtype=torch.uint8, device=flat.device)
    buf[:flat.numel()] = flat
    outs = [torch.empty(n_max, dtype=torch.uint8, device=flat.device) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    res = []
    for (m, n), o in zip(metas, outs):
        res.extend(unpack_blocks(m, o[:n]))
    return res


def all_gather_rows(local, dist, group=None):
    """Full decoded tensor from row shards (the north star's "all-gather decoded shards where
    a consumer needs the full tensor"): rank r holds rows [r·R, (r+1)·R) of a layer, equal
    R on every rank; returns the [world·R, cols] tensor on every rank."""
    import torch
    world = dist.get_world_size(group)
    local = local.contiguous()
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    parts = list(out.chunk(world, dim=0))
    dist.all_gather(parts, local, group=group)
    return out


def link_bytes_per_rank(blocks_per_rank_bytes: float, world: int) -> float:
    """Bytes each rank receives in an all-gather of equal per-rank shards."""
    return blocks_per_rank_bytes * (world - 1)
