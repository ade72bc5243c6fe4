"""EQ_CHUNK_ROW on the GPU: chunks restart at every row start,
so a row of K columns is ⌈K/cs⌉ chunks (4096 + 4096 + 4096 + 2048 for K = 14336).  The
decoders, the encoder and the fused GEMM follow the layout the oracle defines and pins
(tests/test_oracle_codec.py::test_row_chunking_*)."""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq
from test_gpu_parity import DEV, oracle_block_to_gpu, small_layers, table_u16, to_bf16, u16

pytestmark = pytest.mark.gpu
CODECS = [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G]


@pytest.mark.parametrize("codec", CODECS)
@pytest.mark.parametrize("cs", [4096, 1000, 64, 7])
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16])
def test_rowchunk_decode_oracle_streams(codec, cs, out):
    layers = small_layers(seed=2)
    scales = [(o.absmax_scales(W).astype(np.int32) + 1600).astype(np.uint16) for W in layers]
    blk = o.quantize_encode(layers, scales=scales, cs=cs, codec=codec, chunk_mode=o.CHUNK_ROW)
    views = eq.decode_dequant([oracle_block_to_gpu(blk)], out)[0]
    a = 0
    for (r, c), v, S in zip(blk.layer_shapes, views, blk.scales):
        codes = blk.codes[a:a + r * c].reshape(r, c)
        a += r * c
        if out == eq.EQ_OUT_FP8:
            assert (v.view(torch.uint8).cpu().numpy() == codes).all()
        else:
            assert (u16(v) == o.dequant(codes, S)).all()


@pytest.mark.parametrize("codec", CODECS)
@pytest.mark.parametrize("cs", [4096, 333])
def test_rowchunk_encode_byte_identical(codec, cs):
    layers = small_layers(seed=6, shapes=[(12, 14336), (37, 53), (5, 4097)])
    S = [(o.absmax_scales(W).astype(np.int32) + 1500).astype(np.uint16) for W in layers]
    g = eq.quantize_encode([W.to(DEV) for W in layers], scales=to_bf16(np.concatenate(S)), chunk_symbols=cs,
                           codec=codec, chunk_mode=eq.EQ_CHUNK_ROW)
    ref = o.quantize_encode(layers, scales=S, cs=cs, codec=codec, chunk_mode=o.CHUNK_ROW)
    assert g.n_chunks == ref.n_chunks == 12 * ((14336 + cs - 1) // cs) + 37 * ((53 + cs - 1) // cs) + 5 * ((4097 + cs - 1) // cs)
    assert (g.freq.cpu().numpy().view(np.uint16) == table_u16(ref)).all()
    assert (g.chunk_off.cpu().numpy().astype(np.uint32) == ref.chunk_off).all()
    assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == ref.payload
    for v, r in zip(eq.decode_dequant([g], eq.EQ_OUT_BF16)[0], o.decode_dequant(ref)):
        assert (u16(v) == r).all()


@pytest.mark.parametrize("codec", [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G])
@pytest.mark.parametrize("batch", [1, 64])
def test_rowchunk_qmatmul_ragged_k(codec, batch):
    """Fused GEMM on a row-chunked layer whose K is not a multiple of the chunk length:
    K = 14336 at cs = 4096 (4096 + 4096 + 4096 + 2048 per row, Llama-3-8B down_proj) and
    K = 1600 at cs = 1024 (1024 + 576)."""
    shapes = [(128, 14336), (256, 1600)]
    Ws = [eqsynth.weights(r, c, seed=41, layer=0, matrix=m) for m, (r, c) in enumerate(shapes)]
    S = [(o.absmax_scales(W).astype(np.int32) + 128 * 12).astype(np.uint16) for W in Ws]
    for cs in (4096, 1024):
        blk = o.quantize_encode(Ws, scales=S, cs=cs, codec=codec, chunk_mode=o.CHUNK_ROW)
        g = oracle_block_to_gpu(blk)
        What = [d.view(np.int16) for d in o.decode_dequant(blk)]
        for layer, (r, c) in enumerate(shapes):
            x = (torch.randn(batch, c, generator=torch.Generator().manual_seed(layer + batch)) * 0.5).to(torch.bfloat16)
            W64 = torch.from_numpy(What[layer]).view(torch.bfloat16).double().numpy()
            X64 = x.double().numpy()
            ref = X64 @ W64.T
            bound = 1e-4 * (np.abs(X64) @ np.abs(W64).T) + 1e-30
            y = eq.qmatmul(g, layer, x.to(DEV)).cpu().double().numpy()
            assert (np.abs(y - ref) <= bound).all(), (cs, layer, float(np.max(np.abs(y - ref) / bound)))


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
@pytest.mark.parametrize("batch", [1, 64])
def test_qmatmul_escape_heavy_pair_stream(batch, pc):
    """Pair codec with escapes on most steps (uniform bytes: only 15 of the codes are ranked):
    the fused GEMM's escape singles — from the 4 KB symbol table at small batches, by a binary
    search over the cumulative frequencies when the table does not fit 3 CTAs/SM (batch 64) —
    must reproduce the fp64 product of the oracle's dequantised weights."""
    rows, cols = 256, 4096
    s = eqsynth.random_codes_stream(rows * cols, 11, "uniform")
    s = np.where((s & 0x7F) == 0x7F, s ^ 1, s).astype(np.uint8)        # no NaN codes (never produced, R1)
    S = (np.arange(rows, dtype=np.uint16) % 97 + 0x3A00).astype(np.uint16)
    blk = o.encode_codes([s.reshape(rows, cols)], [(rows, cols)], [S], 2048, codec=pc,
                         chunk_mode=o.CHUNK_ROW)
    g = oracle_block_to_gpu(blk)
    W64 = torch.from_numpy(o.dequant(s.reshape(rows, cols), S).view(np.int16)).view(torch.bfloat16).double().numpy()
    x = (torch.randn(batch, cols, generator=torch.Generator().manual_seed(batch)) * 0.5).to(torch.bfloat16)
    X64 = x.double().numpy()
    ref = X64 @ W64.T
    bound = 1e-4 * (np.abs(X64) @ np.abs(W64).T) + 1e-30
    y = eq.qmatmul(g, 0, x.to(DEV)).cpu().double().numpy()
    assert (np.abs(y - ref) <= bound).all(), float(np.max(np.abs(y - ref) / bound))
