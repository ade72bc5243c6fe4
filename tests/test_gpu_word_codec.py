"""GPU parity for the 16-bit-word rANS codec (EQ_CODEC_WORD, reading R14) through
the C-ABI: decode of oracle-encoded streams (symbols and bf16 bit-exact), GPU encode
byte-identical to the oracle, Alg. 1 end to end, integrity checks, the host-buffer path.
"""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq
from test_gpu_parity import DEV, RAGGED, oracle_block_to_gpu, small_layers, to_bf16, u16

pytestmark = pytest.mark.gpu
W16 = o.CODEC_WORD


@pytest.mark.parametrize("cs", [262144, 4096, 1000, 64, 7, 1])
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16])
def test_word_decode_oracle_streams(cs, out):
    layers = small_layers()
    scales = [o.absmax_scales(W) for W in layers]
    scales[2] = (scales[2].astype(np.int32) + 1700).astype(np.uint16)       # ~2-bit regime rows
    scales[4] = (scales[4].astype(np.int32) + 2000).astype(np.uint16)       # near-zero entropy rows
    blk = o.quantize_encode(layers, scales=scales, cs=cs, codec=W16)
    views = eq.decode_dequant([oracle_block_to_gpu(blk)], out)[0]
    a = 0
    for (r, c), v, S in zip(blk.layer_shapes, views, blk.scales):
        codes = blk.codes[a:a + r * c].reshape(r, c)
        a += r * c
        if out == eq.EQ_OUT_FP8:
            assert (v.view(torch.uint8).cpu().numpy() == codes).all()
        else:
            assert (u16(v) == o.dequant(codes, S)).all()


@pytest.mark.parametrize("kind", ["uniform", "subset2", "single", "skewed"])
def test_word_decode_extreme_streams(kind):
    """Table extremes: 8 bits/symbol (one word every second symbol), a single symbol
    (f = M, no words at all), two symbols."""
    n = 64 * 4096
    s = eqsynth.random_codes_stream(n, 3, kind)
    s = np.where(s == 0x7F, 0x7E, np.where(s == 0xFF, 0xFE, s)).astype(np.uint8)   # no NaN codes
    blk = o.encode_codes([s.reshape(64, 4096)], [(64, 4096)], [np.full(64, 0x3F80, np.uint16)], 4096,
                         codec=W16)
    v = eq.decode_dequant([oracle_block_to_gpu(blk)], eq.EQ_OUT_FP8)[0][0]
    assert (v.view(torch.uint8).cpu().numpy().reshape(-1) == s).all()


def test_word_decode_many_blocks_one_launch():
    blocks, refs = [], []
    for b in range(5):
        layers = small_layers(seed=10 + b, shapes=[(32, 256), (7, 96), (48, 512)])
        scales = [(o.absmax_scales(W).astype(np.int32) + 128 * (6 + b)).astype(np.uint16) for W in layers]
        ob = o.quantize_encode(layers, scales=scales, cs=512, codec=W16)
        blocks.append(oracle_block_to_gpu(ob))
        refs.append(o.decode_dequant(ob))
    views = eq.decode_dequant(blocks, eq.EQ_OUT_BF16)
    for vb, rb in zip(views, refs):
        for v, r in zip(vb, rb):
            assert (u16(v) == r).all()


def test_word_mixed_codecs_rejected():
    layers = small_layers(shapes=[(16, 256)])
    a = oracle_block_to_gpu(o.quantize_encode(layers, lam=None, cs=256, codec=W16))
    b = oracle_block_to_gpu(o.quantize_encode(layers, lam=None, cs=256))
    with pytest.raises(eq.EqError) as ei:
        eq.decode_dequant([a, b], eq.EQ_OUT_FP8)
    assert ei.value.status == eq.EQ_ERR_ARG


def test_word_decode_detects_corruption_and_truncation():
    layers = small_layers(shapes=[(64, 512)])
    blk = o.quantize_encode(layers, lam=None, cs=512, codec=W16)
    g = oracle_block_to_gpu(blk)
    d = eq.Decoder([g], eq.EQ_OUT_FP8)
    d()
    d.check()
    a, b = int(blk.chunk_off[3]), int(blk.chunk_off[4])
    g.payload[(a + b) // 2] ^= 0x5A
    d.err.zero_()
    d()
    with pytest.raises(eq.EqError) as ei:
        d.check()
    assert ei.value.status == eq.EQ_ERR_CORRUPT
    g.payload[(a + b) // 2] ^= 0x5A
    # a chunk boundary moved by one word: both neighbours fail the length check
    g.chunk_off[5] += 2
    d.err.zero_()
    d()
    with pytest.raises(eq.EqError) as ei:
        d.check()
    assert ei.value.status == eq.EQ_ERR_CORRUPT
    g.chunk_off[5] -= 2
    g.chunk_off[-1] = blk.chunk_off[-1] + 1000
    d.err.zero_()
    d()
    with pytest.raises(eq.EqError) as ei:
        d.check()
    assert ei.value.status == eq.EQ_ERR_TRUNCATED


@pytest.mark.parametrize("cs", [4096, 333, 1])
def test_word_rans_encode_byte_identical(cs):
    layers = small_layers()
    scales = [(o.absmax_scales(W).astype(np.int32) + 1500).astype(np.uint16) for W in layers]
    blk = o.quantize_encode(layers, scales=scales, cs=cs, codec=W16)
    g = eq.rans_encode(torch.from_numpy(blk.codes).to(DEV), blk.layer_shapes,
                       torch.from_numpy(blk.freq.view(np.int16).copy()).to(DEV), chunk_symbols=cs, codec=W16)
    assert g.payload_bytes == len(blk.payload)
    assert (g.chunk_off.cpu().numpy().astype(np.uint32) == blk.chunk_off).all()
    assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == blk.payload


@pytest.mark.parametrize("fmt", [eq.EQ_FMT_E4M3, eq.EQ_FMT_INT8])
def test_word_quantize_encode_end_to_end(fmt):
    """Alg. 1 on the GPU with the word codec, given the oracle's scales: stream, offsets and
    table byte-identical; decode + dequant identical to the oracle's."""
    layers = small_layers(seed=3)
    S = [o.search(W, 150.0, fmt=fmt)[0] if i % 2 == 0 else o.absmax_scales(W, fmt) for i, W in enumerate(layers)]
    g = eq.quantize_encode([W.to(DEV) for W in layers], scales=to_bf16(np.concatenate(S)), chunk_symbols=1000,
                           format=fmt, codec=W16)
    ref = o.quantize_encode(layers, scales=S, cs=1000, fmt=fmt, codec=W16)
    assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == ref.payload
    assert (g.freq.cpu().numpy().view(np.uint16) == ref.freq).all()
    for v, r in zip(eq.decode_dequant([g], eq.EQ_OUT_BF16)[0], o.decode_dequant(ref)):
        assert (u16(v) == r).all()


def test_word_host_buffer_e2e_decode():
    layers = small_layers(seed=8, shapes=[(64, 256), (32, 512)])
    g = eq.quantize_encode([W.to(DEV) for W in layers], lam=80.0, codec=W16)
    hb = eq.HostBlocks([g], eq.EQ_OUT_BF16)
    arena = hb.decode()
    dev = eq.Decoder([g], eq.EQ_OUT_BF16)
    dev()
    dev.check()
    assert torch.equal(arena[:dev.total], dev.arena[:dev.total].cpu())


def test_word_rate_vs_byte_codec_at_two_bits():
    """Same codes, both codecs: the word codec's payload stays within 1.02x of n·Ĥ/8 with
    offsets (north_star) and within 0.5 % of the byte codec's."""
    W = eqsynth.weights(512, 4096, seed=6)
    gw = eq.quantize_encode([W.to(DEV)], lam=230.0, codec=W16)
    gb = eq.quantize_encode([W.to(DEV)], scales=gw.scales, codec=eq.EQ_CODEC_BYTE)
    codes, hist = eq.quantize_hist(W.to(DEV), gw.scales)
    H = o.entropy(hist.cpu().numpy().astype(np.uint64))
    assert gw.payload_bytes + 4 * (gw.n_chunks + 1) <= 1.02 * W.numel() * H / 8
    assert abs(gw.payload_bytes - gb.payload_bytes) <= 0.005 * gb.payload_bytes


def test_word_decode_max_chunk_full_rows():
    """The largest chunk SPEC allows (262144 symbols) on rows of 14336 (a chunk spans
    rows, so the per-group scale switch inside a chunk is exercised) and 8 such layers."""
    shapes = [(32, 14336)] * 2 + [(64, 4096)]
    layers = [eqsynth.weights(r, c, seed=21, layer=1, matrix=m) for m, (r, c) in enumerate(shapes)]
    S = [(o.absmax_scales(W).astype(np.int32) + 1600).astype(np.uint16) for W in layers]
    blk = o.quantize_encode(layers, scales=S, cs=262144, codec=W16)
    g = oracle_block_to_gpu(blk)
    for v, r in zip(eq.decode_dequant([g], eq.EQ_OUT_BF16)[0], o.decode_dequant(blk)):
        assert (u16(v) == r).all()


@pytest.mark.parametrize("codec", [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G])
def test_decode_under_random_corruption_matches_oracle_verdicts(codec):
    """Fuzz: random byte flips in the payload.  The GPU decoder never faults; every chunk the
    oracle rejects makes the launch report an error; when the oracle accepts every chunk of a
    corrupted block (a flip can yield another valid stream), the GPU output equals the
    oracle's decode of the same corrupted bytes."""
    layers = small_layers(seed=40, shapes=[(32, 512), (16, 1024)])
    S = [(o.absmax_scales(W).astype(np.int32) + 1600).astype(np.uint16) for W in layers]
    blk = o.quantize_encode(layers, scales=S, cs=512, codec=codec)
    rng = np.random.default_rng(codec)
    base = bytearray(blk.payload)
    accepted = rejected = 0
    for trial in range(40):
        data = bytearray(base)
        for _ in range(int(rng.integers(1, 4))):
            data[int(rng.integers(0, len(data)))] ^= int(rng.integers(1, 256))
        cb = o.OracleBlock(blk.layer_shapes, blk.scales, blk.freq, blk.hist, bytes(data), blk.chunk_off,
                           blk.chunk_symbols, None, blk.fmt, codec, blk.pair)
        try:
            ref = o.decode_dequant(cb)
        except ValueError:
            ref = None
        g = oracle_block_to_gpu(cb)
        d = eq.Decoder([g], eq.EQ_OUT_BF16)
        d()
        if ref is None:
            with pytest.raises(eq.EqError) as ei:
                d.check()
            assert ei.value.status in (eq.EQ_ERR_CORRUPT, eq.EQ_ERR_TRUNCATED)
            rejected += 1
        else:
            d.check()
            for v, r in zip(d.views()[0], ref):
                assert (u16(v) == r).all()
            accepted += 1
    assert rejected > 20
