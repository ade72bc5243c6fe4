"""NCCL path of the block exchange on the one GPU a gpurun box has: a
world-size-1 NCCL group runs all_gather_blocks / all_gather_rows through the same code the
multi-GPU case uses, and the gathered blocks decode bit-exactly on the device."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, q):
    import torch.distributed as dist

    import eqsynth
    import oracle as o
    import paper_2601_22787_b200 as eq
    from paper_2601_22787_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    Ws = [eqsynth.weights(r, c, seed=9, layer=0, matrix=m) for m, (r, c) in enumerate([(64, 512), (32, 1024)])]
    blocks = [eq.quantize_encode([W.to(dev) for W in Ws], lam=120.0, codec=c) for c in (eq.EQ_CODEC_WORD, eq.EQ_CODEC_BYTE)]
    got = shard.all_gather_blocks(blocks, dist)
    ok = len(got) == 2
    for a, b in zip(blocks, got):
        ok &= b.payload.is_cuda and b.codec == a.codec and b.payload_bytes == a.payload_bytes
        ok &= torch.equal(a.payload[:a.payload_bytes], b.payload[:b.payload_bytes])
        va, vb = eq.decode_dequant([a], eq.EQ_OUT_BF16)[0], eq.decode_dequant([b], eq.EQ_OUT_BF16)[0]
        ok &= all(torch.equal(x.view(torch.int16), y.view(torch.int16)) for x, y in zip(va, vb))
    full = eq.decode_dequant([got[0]], eq.EQ_OUT_BF16)[0][0]
    ok &= torch.equal(shard.all_gather_rows(full, dist), full)
    dist.destroy_process_group()
    q.put(bool(ok))


def test_nccl_block_all_gather_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_port(), q))
    p.start()
    ok = q.get(timeout=300)
    p.join(60)
    assert p.exitcode == 0 and ok
