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
        assert sorted(flat) == list(range(blocks))           # one layer set split
    for rank, _, m, v in res:
        assert m == 15.0                                     # MAX over ranks
        assert v == pytest.approx(1e9 * world * 4 / 0.015 / 1e9)


def test_single_process_identity_and_errors():
    assert shard.max_over_ranks(3.5) == 3.5
    assert shard.layer_ids(0, 1, 3) == [0, 1, 2]
    with pytest.raises(ValueError):
        shard.layer_ids(2, 2, 3)
