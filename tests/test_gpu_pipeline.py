"""NEXT row 2 (block-pipelined inference arena): the pipelined forward (S slots, decode of
upcoming blocks on a side stream) equals the forward on the oracle's decoded weights."""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq
from paper_2601_22787_b200.pipeline import BlockPipeline, llama_block_forward

pytestmark = pytest.mark.gpu

SHAPES = [(256, 256), (64, 256), (64, 256), (256, 256), (512, 256), (512, 256), (256, 512)]


def test_pipeline_matches_oracle_weights():
    dev = torch.device("cuda")
    blocks, ref_blocks = [], []
    for lid in range(5):
        Ws = [eqsynth.weights(r, c, seed=7, layer=lid, matrix=m) for m, (r, c) in enumerate(SHAPES)]
        S = [(o.absmax_scales(W).astype(np.int32) + 128 * 11).astype(np.uint16) for W in Ws]
        ob = o.quantize_encode(Ws, scales=S)
        ref_blocks.append([torch.from_numpy(d.view(np.int16)).view(torch.bfloat16).to(dev) for d in o.decode_dequant(ob)])
        sc = torch.from_numpy(np.concatenate(S).view(np.int16)).view(torch.bfloat16).to(dev)
        blocks.append(eq.quantize_encode([W.to(dev) for W in Ws], scales=sc, codec=eq.EQ_CODEC_BYTE))
    x0 = (torch.arange(4 * 256, device=dev, dtype=torch.float32).reshape(4, 256).sin() * 0.1).to(torch.bfloat16)
    ref = x0
    for views in ref_blocks:
        ref = llama_block_forward(views, ref)
    for slots, group in ((1, 1), (2, 1), (3, 1), (2, 2), (1, 5), (2, 3)):
        pipe = BlockPipeline(blocks, slots=slots, group=group)
        y = pipe.run(lambda k, views, x: llama_block_forward(views, x), x0)
        torch.cuda.synchronize()
        pipe.check()
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16)), slots


def test_fused_gemm_forward_matches_dense_forward_on_oracle_weights():
    """The decode-fused forward (four eq_qmatmul_group launches per block, weights never
    materialised) against the dense forward on the oracle's dequantised weights: the same
    dataflow, so they differ only by fp32 accumulation order (and the bf16 roundings that
    follows from it)."""
    from paper_2601_22787_b200.pipeline import llama_block_forward_fused
    dev = torch.device("cuda")
    shapes = [(256, 256), (128, 256), (128, 256), (256, 256), (512, 256), (512, 256), (256, 512)]
    x0 = (torch.arange(8 * 256, device=dev, dtype=torch.float32).reshape(8, 256).cos() * 0.2).to(torch.bfloat16)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(1 << 22, dtype=torch.uint8, device=dev)
    for codec in (o.CODEC_PAIR_G, o.CODEC_PAIR, o.CODEC_WORD):
        x_ref = x_fused = x0
        for lid in range(3):
            Ws = [eqsynth.weights(r, c, seed=9, layer=lid, matrix=m) for m, (r, c) in enumerate(shapes)]
            S = [(o.absmax_scales(W).astype(np.int32) + 128 * 11).astype(np.uint16) for W in Ws]
            ob = o.quantize_encode(Ws, scales=S, cs=128, codec=codec, chunk_mode=o.CHUNK_ROW)
            views = [torch.from_numpy(d.view(np.int16)).view(torch.bfloat16).to(dev) for d in o.decode_dequant(ob)]
            sc = torch.from_numpy(np.concatenate(S).view(np.int16)).view(torch.bfloat16).to(dev)
            blk = eq.quantize_encode([W.to(dev) for W in Ws], scales=sc, codec=codec, chunk_symbols=128,
                                     chunk_mode=eq.EQ_CHUNK_ROW)
            x_ref = llama_block_forward(views, x_ref)
            x_fused = llama_block_forward_fused(blk, x_fused, err, ws)
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        d = (x_fused.float() - x_ref.float()).abs()
        assert float(d.max()) <= 2e-2 * float(x_ref.float().abs().max()), (codec, float(d.max()))
