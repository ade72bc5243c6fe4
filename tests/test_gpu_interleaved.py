"""EQ_CHUNK_INTERLEAVED (R17) on the GPU: the encoder's payload, offsets and table equal
the oracle's byte for byte; k_decode_p's bf16 / FP8 output equals the oracle's decode; argument
validation."""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq
from test_gpu_parity import DEV, oracle_block_to_gpu, small_layers, table_u16, to_bf16, u16

pytestmark = pytest.mark.gpu
IL = eq.EQ_CHUNK_INTERLEAVED


def _layers(shapes, seed):
    return [eqsynth.weights(r, c, seed=seed, layer=0, matrix=m) for m, (r, c) in enumerate(shapes)]


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
@pytest.mark.parametrize("cs", [4096, 256, 32])
def test_interleaved_encode_byte_identical_and_decode(cs, pc):
    """Whole super-chunks plus ragged tails of plain chunks (24·704 = 16896 symbols: at cs 256,
    2 super-chunks of 8192 and a 512-symbol tail)."""
    shapes = [(64, 4096), (24, 704), (48, 1024)]
    layers = _layers(shapes, 21)
    S = [(o.absmax_scales(W).astype(np.int32) + 128 * 12).astype(np.uint16) for W in layers]
    ref = o.quantize_encode(layers, scales=S, cs=cs, codec=pc, chunk_mode=o.CHUNK_INTERLEAVED)
    g = eq.quantize_encode([W.to(DEV) for W in layers], scales=to_bf16(np.concatenate(S)), chunk_symbols=cs,
                           codec=pc, chunk_mode=IL)
    assert g.n_chunks == ref.n_chunks
    assert (g.freq.cpu().numpy().view(np.uint16) == table_u16(ref)).all()
    assert (g.chunk_off.cpu().numpy().astype(np.uint32) == ref.chunk_off).all()
    assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == ref.payload
    for v, r in zip(eq.decode_dequant([g], eq.EQ_OUT_BF16)[0], o.decode_dequant(ref)):
        assert (u16(v) == r).all()
    stream = o.decode_block(ref)
    a = 0
    for v, (r, c) in zip(eq.decode_dequant([g], eq.EQ_OUT_FP8)[0], shapes):
        assert (v.view(torch.uint8).cpu().numpy().reshape(-1) == stream[a:a + r * c]).all()
        a += r * c


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
@pytest.mark.parametrize("cs", [4096, 64, 32])
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16])
def test_interleaved_decode_oracle_streams(cs, out, pc):
    """Streams written by the oracle's encoder (independent of the GPU one); shapes whose symbol
    counts end in partial super-chunks and in a tail shorter than one group."""
    layers = small_layers(seed=9, shapes=[(16, 4096), (3, 4112), (64, 64), (1, 16)])
    scales = [(o.absmax_scales(W).astype(np.int32) + 1600).astype(np.uint16) for W in layers]
    blk = o.quantize_encode(layers, scales=scales, cs=cs, codec=pc, chunk_mode=o.CHUNK_INTERLEAVED)
    views = eq.decode_dequant([oracle_block_to_gpu(blk)], out)[0]
    a = 0
    for (r, c), v, S in zip(blk.layer_shapes, views, blk.scales):
        codes = blk.codes[a:a + r * c].reshape(r, c)
        a += r * c
        if out == eq.EQ_OUT_FP8:
            assert (v.view(torch.uint8).cpu().numpy() == codes).all()
        else:
            assert (u16(v) == o.dequant(codes, S)).all()


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
def test_interleaved_decode_many_blocks_one_launch_vs_layer_mode(pc):
    """Three blocks in one launch: the interleaved streams decode to the same weights as the
    layer-chunked streams of the same codes (the layout is a permutation of chunk membership)."""
    blocks_il, blocks_l = [], []
    for b in range(3):
        layers = _layers([(128, 1024), (64, 2048)], 30 + b)
        S = [(o.absmax_scales(W).astype(np.int32) + 128 * 13).astype(np.uint16) for W in layers]
        sc = to_bf16(np.concatenate(S))
        Ws = [W.to(DEV) for W in layers]
        blocks_il.append(eq.quantize_encode(Ws, scales=sc, chunk_symbols=64, codec=pc, chunk_mode=IL))
        blocks_l.append(eq.quantize_encode(Ws, scales=sc, chunk_symbols=64, codec=pc))
    a = eq.decode_dequant(blocks_il, eq.EQ_OUT_BF16)
    b = eq.decode_dequant(blocks_l, eq.EQ_OUT_BF16)
    for va, vb in zip(a, b):
        for x, y in zip(va, vb):
            assert torch.equal(x.view(torch.int16), y.view(torch.int16))


def test_interleaved_argument_validation():
    W = eqsynth.weights(32, 512, seed=3).to(DEV)
    with pytest.raises(eq.EqError) as e:                       # word codec: not decoded by R17 kernels
        eq.quantize_encode([W], lam=100.0, codec=eq.EQ_CODEC_WORD, chunk_mode=IL)
    assert e.value.status == eq.EQ_ERR_ARG
    with pytest.raises(eq.EqError) as e:                       # chunk length not a multiple of 32
        eq.quantize_encode([W], lam=100.0, chunk_symbols=48, codec=eq.EQ_CODEC_PAIR, chunk_mode=IL)
    assert e.value.status == eq.EQ_ERR_ARG
    W2 = eqsynth.weights(32, 520, seed=3).to(DEV)              # cols % 16 != 0
    with pytest.raises(eq.EqError) as e:
        eq.quantize_encode([W2], lam=100.0, codec=eq.EQ_CODEC_PAIR, chunk_mode=IL)
    assert e.value.status == eq.EQ_ERR_SHAPE
    blk = eq.quantize_encode([eqsynth.weights(128, 512, seed=4).to(DEV)], lam=100.0, chunk_symbols=512,
                             codec=eq.EQ_CODEC_PAIR, chunk_mode=IL)
    with pytest.raises(eq.EqError):                            # the fused GEMM needs row-contiguous chunks
        eq.qmatmul(blk, 0, torch.zeros(1, 512, dtype=torch.bfloat16, device=DEV))


def test_mixed_chunk_lengths_in_one_launch():
    """The bench's tail blocks: blocks of different chunk lengths in ONE
    eq_decode_dequant launch, each block's bf16 layers equal to the oracle's decode."""
    shapes = [(64, 256), (32, 512), (16, 1024)]
    gpu_blocks, refs = [], []
    for b, cs in enumerate((64, 32, 64, 128)):
        layers = _layers(shapes, 40 + b)
        S = [(o.absmax_scales(W).astype(np.int32) + 128 * 11).astype(np.uint16) for W in layers]
        refs.append(o.quantize_encode(layers, scales=S, cs=cs, codec=o.CODEC_PAIR_G, chunk_mode=o.CHUNK_INTERLEAVED))
        gpu_blocks.append(eq.quantize_encode([W.to(DEV) for W in layers], scales=to_bf16(np.concatenate(S)),
                                             chunk_symbols=cs, codec=eq.EQ_CODEC_PAIR_G, chunk_mode=IL))
    views = eq.decode_dequant(gpu_blocks, eq.EQ_OUT_BF16)
    for vb, ref in zip(views, refs):
        for v, r in zip(vb, o.decode_dequant(ref)):
            assert (u16(v) == r).all()
