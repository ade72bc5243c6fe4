"""world_size-2 gloo tests of the multi-GPU host logic (block sharding, MAX-over-ranks
timing, whole-job aggregation) — runs on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_22787_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, blocks, scaling, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = shard.layer_ids(rank, world, blocks, scaling)
    gathered = [None] * world
    dist.all_gather_object(gathered, ids)
    elapsed = 10.0 + 5.0 * rank                      # rank 1 is the slow one
    m = shard.max_over_ranks(elapsed, dist)
    v = shard.aggregate_gbs(1e9, world, 4, m)
    dist.barrier()
    q.put((rank, gathered, m, v))
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_two_rank_sharding_and_timing(scaling):
    world, blocks = 2, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, blocks, scaling, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    gathered = res[0][1]
    assert res[1][1] == gathered
    flat = [i for ids in gathered for i in ids]
    assert len(flat) == len(set(flat))                       # disjoint shards
    if scaling == "weak":
        assert flat == list(range(world * blocks))           # each rank its own layer set
        assert all(len(ids) == blocks for ids in gathered)
    else:
        assert flat == list(range(blocks))                   # one layer set, contiguous ranges
        assert [len(ids) for ids in gathered] == [4, 3]      # 7 blocks: the first rank takes the extra
    for rank, _, m, v in res:
        assert m == 15.0                                     # MAX over ranks
        assert v == pytest.approx(1e9 * world * 4 / 0.015 / 1e9)


def test_single_process_identity_and_errors():
    assert shard.max_over_ranks(3.5) == 3.5
    assert shard.layer_ids(0, 1, 3) == [0, 1, 2]
    # 32 Llama-3-8B blocks over G = 2, 4, 8 ranks -> contiguous 16 / 8 / 4-block ranges
    for G in (2, 4, 8):
        parts = [shard.layer_ids(r, G, 32) for r in range(G)]
        assert [i for p in parts for i in p] == list(range(32))
        assert all(p == list(range(r * 32 // G, (r + 1) * 32 // G)) for r, p in enumerate(parts))
    with pytest.raises(ValueError):
        shard.layer_ids(2, 2, 3)


def _gather_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np

    import eqsynth
    import oracle as o
    import paper_2601_22787_b200 as eq
    # rank r holds compressed blocks of layers 2r, 2r+1 (CPU tensors stand in for device memory)
    mine = []
    for lid in (2 * rank, 2 * rank + 1):
        Ws = [eqsynth.weights(r_, c, seed=5, layer=lid, matrix=m) for m, (r_, c) in enumerate([(32, 256), (16, 384)])]
        ob = o.quantize_encode(Ws, lam=None, cs=512, codec=o.CODEC_WORD if lid % 2 else o.CODEC_BYTE)
        cap = len(ob.payload) + 256
        pay = torch.zeros(cap, dtype=torch.uint8)
        pay[:len(ob.payload)] = torch.frombuffer(bytearray(ob.payload), dtype=torch.uint8)
        mine.append(eq.Block(pay, len(ob.payload), torch.from_numpy(ob.chunk_off.astype(np.int64).astype(np.int32)),
                             torch.from_numpy(ob.freq.view(np.int16).copy()),
                             torch.from_numpy(np.concatenate(ob.scales).view(np.int16)).view(torch.bfloat16),
                             list(ob.layer_shapes), 512, {"layer": lid}, ob.fmt, ob.codec))
    allb = shard.all_gather_blocks(mine, dist)
    # decoded-row all-gather: rank r holds rows [4r, 4r+4) of an 8 x 6 tensor
    full = torch.arange(48, dtype=torch.float32).view(8, 6)
    rows = shard.all_gather_rows(full[4 * rank:4 * rank + 4].clone(), dist)
    summary = []
    for b in allb:
        ob = o.OracleBlock(b.shapes, [], b.freq.numpy().view(np.uint16), None,
                           b.payload[:b.payload_bytes].numpy().tobytes(), b.chunk_off.numpy().astype(np.uint32),
                           b.chunk_symbols, None, b.format, b.codec)
        stream = o.decode_block(ob)
        summary.append((b.meta["layer"], b.codec, int(stream.sum()), b.payload_bytes,
                        bytes(b.scales.view(torch.int16).numpy().tobytes())))
    q.put((rank, summary, bool(torch.equal(rows, full))))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_compressed_block_all_gather():
    """Every rank ends with every rank's compressed blocks, byte-identical (streams decode
    with the oracle to the same symbols on both ranks), plus the decoded-row all-gather."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    (_, s0, ok0), (_, s1, ok1) = res
    assert ok0 and ok1
    assert s0 == s1
    assert [t[0] for t in s0] == [0, 1, 2, 3]                 # rank-major order
    assert [t[1] for t in s0] == [0, 1, 0, 1]                 # codecs travel with the blocks
