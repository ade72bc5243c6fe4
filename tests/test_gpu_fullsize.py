"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration.

Config 3: the 32-block Llama-3-8B-shaped layer set is encoded on the GPU (search at the
bench's λ, word codec as in the bench and the byte codec) and decoded in ONE
eq_decode_dequant launch into the bf16 arena.  The oracle
recomputes sampled rows one by one from the INPUT weights (its own search, quantiser and
dequantiser) and must equal the decoded rows bit for bit (rows whose GPU scale is a
documented near-tie of the oracle's objective are checked for optimality instead).
Every symbol: the oracle's own decoder (threaded, the bench's CPU-baseline helper) decodes
every chunk of all 32 blocks and its bf16 output must equal the GPU arena of the bench's
launch bit for bit (~7.0 G symbols per codec).  Encode at full size: for blocks 0, 15 and 31
the oracle re-runs Alg. 1 l.3-5 from the INPUT weights with the GPU's scales (the search is
checked separately on sampled rows) and must reproduce the GPU's table, offsets and payload
byte for byte.  Properties checked at full size: coded size ≤ 1.02× the histogram entropy,
Shannon's bound, effective rate near the target.
Configs 2 and 5: every symbol of the 16-block Llama-3.2-1B set and of one whole Llama-3-70B block
against the oracle's decoder, and a sampled block's encode against the oracle's.
"""
import os

import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq

pytestmark = pytest.mark.gpu
LAM = 230.2          # the bench's calibrated λ for 2.0 bits (bench.py DEFAULT_LAMBDA)


def u16(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def test_eqsynth_bit_identical_on_cuda():
    for dist in eqsynth.DISTS:
        a = eqsynth.weights(129, 1000, seed=4, layer=3, matrix=2, dist=dist)
        b = eqsynth.weights(129, 1000, seed=4, layer=3, matrix=2, dist=dist, device="cuda")
        assert torch.equal(a.view(torch.int16), b.cpu().view(torch.int16)), dist


@pytest.fixture(scope="module", params=[(eq.EQ_CODEC_PAIR_G, eq.EQ_CHUNK_INTERLEAVED),
                                        (eq.EQ_CODEC_PAIR, eq.EQ_CHUNK_LAYER),
                                        (eq.EQ_CODEC_WORD, eq.EQ_CHUNK_LAYER), (eq.EQ_CODEC_BYTE, eq.EQ_CHUNK_LAYER)],
                ids=["pairg-il", "pair", "word", "byte"])
def layer_set(request):
    """The bench's layer set in its encoding (R18 pair codec, R17 interleaved chunks), the
    pair codec of R15 with layer chunks, the word codec (R14) and SPEC's byte codec (R9)."""
    codec, mode = request.param
    dev = torch.device("cuda")
    blocks, kept = [], {}
    scratch = None
    for lid in range(32):
        Ws = eqsynth.block_weights("llama-3-8b", lid, device=dev)
        if scratch is None:
            scratch = torch.empty(eq.encode_bounds(Ws, codec=eq.EQ_CODEC_BYTE)[2], dtype=torch.uint8, device=dev)
        blocks.append(eq.quantize_encode(Ws, lam=LAM, scratch=scratch, codec=codec, chunk_mode=mode))
        if lid in (0, 15, 31):
            kept[lid] = [W.cpu() for W in Ws]          # the INPUT weights, for the oracle
        del Ws
    del scratch
    torch.cuda.empty_cache()
    return blocks, kept


def _host_block(b):
    """Host copies of a GPU block for the oracle: payload, offsets, table, scales."""
    payload = b.payload.cpu().numpy()
    off = b.chunk_off.cpu().numpy().astype(np.uint32)
    table = b.freq.cpu().numpy().view(np.uint16)
    pair = None
    if b.codec in eq.PAIR_CODECS:
        pair = o.PairTable(table.view(np.uint8)[968:984].copy(), int(table[482]), table[256:481].copy(),
                           int(table[481]))
    return payload, off, table, pair, u16(b.scales)


def test_config3_every_symbol_matches_oracle_decode(layer_set):
    """All 32 blocks, every chunk: the oracle's decoder on the host cores vs the GPU arena of
    the bench's single launch, bf16 bit for bit (Alg. 2 l.1-2)."""
    blocks, _ = layer_set
    dec = eq.Decoder(blocks, eq.EQ_OUT_BF16)
    dec()
    dec.check()
    views = dec.views()
    threads = os.cpu_count() or 1
    total = 0
    for b, vb in zip(blocks, views):
        payload, off, table, pair, scales = _host_block(b)
        k0 = r0 = 0
        for (r, c), v in zip(b.shapes, vb):
            nk = (r * c + b.chunk_symbols - 1) // b.chunk_symbols
            ref = o.decode_dequant_layer_mt(payload, off[k0:k0 + nk + 1], b.chunk_symbols, r, c, scales[r0:r0 + r],
                                            table[:256], threads, b.codec, pair, b.chunk_mode)
            got = u16(v).reshape(r, c)
            assert np.array_equal(ref, got), (b.codec, r, c, int(np.count_nonzero(ref != got)))
            total += r * c
            k0 += nk
            r0 += r
    assert total == 32 * 218103808


def test_config3_full_block_encode_matches_oracle(layer_set):
    """Blocks 0, 15, 31 at full size: the oracle quantises the INPUT weights with the GPU's
    scales and entropy-codes them (its own table rules R8/R15 and coder): table, offsets and
    payload equal the GPU's byte for byte (Alg. 1 l.3-5)."""
    blocks, kept = layer_set
    for lid, Ws in kept.items():
        b = blocks[lid]
        _, off, table, _, scales = _host_block(b)
        S, r0 = [], 0
        for (r, _) in b.shapes:
            S.append(scales[r0:r0 + r])
            r0 += r
        ref = o.quantize_encode(Ws, scales=S, cs=b.chunk_symbols, codec=b.codec, chunk_mode=b.chunk_mode)
        want = np.zeros_like(table)
        want[:256] = ref.freq
        if b.codec in eq.PAIR_CODECS:
            want[256:481] = ref.pair.pf
            want[481] = ref.pair.fesc
            want[482] = ref.pair.K
            want.view(np.uint8)[968:984] = ref.pair.rank_code
        assert np.array_equal(table, want), lid
        assert np.array_equal(off, np.asarray(ref.chunk_off, dtype=np.uint32)), lid
        assert b.payload_bytes == len(ref.payload), lid
        assert b.payload[:b.payload_bytes].cpu().numpy().tobytes() == ref.payload, lid


def test_config3_decode_sampled_rows_match_oracle(layer_set):
    blocks, kept = layer_set
    dec = eq.Decoder(blocks, eq.EQ_OUT_BF16)            # the bench's single launch
    dec()
    dec.check()
    views = dec.views()
    rng = np.random.default_rng(0)
    checked = near = 0
    for lid, Ws in kept.items():
        for m, W in enumerate(Ws):
            Wb = o._u16(W)
            M = Wb.shape[0]
            rows = sorted(set(rng.integers(0, M, 2).tolist()) | {0, M - 1})
            S_or, f_or = o.search(Wb, LAM, rows=rows)
            start = sum(r for r, _ in blocks[lid].shapes[:m])
            S_gpu = u16(blocks[lid].scales[start:start + M])
            out = u16(views[lid][m])
            for r in rows:
                if S_gpu[r] != S_or[r]:
                    first, f = o.row_objectives(Wb, r, LAM)
                    assert f[int(S_gpu[r]) - first] <= f.min() * (1 + 1e-9), (lid, m, r)
                    near += 1
                    continue
                ref = o.dequant(o.quantize(Wb[r:r + 1], S_or[r:r + 1]), S_or[r:r + 1])[0]
                assert (out[r] == ref).all(), (lid, m, r)
                checked += 1
    assert checked >= 50 and near <= 2


def test_config3_lossless_and_rate_properties(layer_set):
    blocks, _ = layer_set
    dec = eq.Decoder(blocks, eq.EQ_OUT_FP8)
    dec()
    dec.check()
    v8 = dec.views()
    n = comp = 0
    for b, vs in zip(blocks[::8], v8[::8]):
        codes = torch.cat([v.reshape(-1).view(torch.uint8) for v in vs])
        hist = torch.bincount(codes.long(), minlength=256).cpu().numpy()
        p = hist[hist > 0] / hist.sum()
        H = float(-(p * np.log2(p)).sum())
        coded = b.payload_bytes + 4 * (b.n_chunks + 1)
        assert coded <= 1.02 * b.n_params * H / 8                     # north_star 1.02×
        assert 8 * b.payload_bytes >= b.n_params * H * (1 - 1e-3)    # Shannon
        # re-encoding the decoded codes with the same table reproduces the payload exactly
        again = eq.rans_encode(codes, b.shapes, b.freq, codec=b.codec, chunk_mode=b.chunk_mode)
        assert again.payload_bytes == b.payload_bytes
        assert torch.equal(again.payload[:again.payload_bytes], b.payload[:b.payload_bytes])
        n += b.n_params
        comp += b.compressed_bytes()
    assert 1.9 < 8 * comp / n < 2.1


def _decode_all_vs_oracle(blocks):
    """Every symbol of one eq_decode_dequant launch over ``blocks`` against the oracle's
    threaded decoder, bf16 bit for bit; returns the number of symbols checked."""
    dec = eq.Decoder(blocks, eq.EQ_OUT_BF16)
    dec()
    dec.check()
    views = dec.views()
    threads = os.cpu_count() or 1
    total = 0
    for b, vb in zip(blocks, views):
        payload, off, table, pair, scales = _host_block(b)
        k0 = r0 = 0
        for (r, c), v in zip(b.shapes, vb):
            nk = (r * c + b.chunk_symbols - 1) // b.chunk_symbols
            ref = o.decode_dequant_layer_mt(payload, off[k0:k0 + nk + 1], b.chunk_symbols, r, c, scales[r0:r0 + r],
                                            table[:256], threads, b.codec, pair, b.chunk_mode)
            assert np.array_equal(ref, u16(v).reshape(r, c)), (b.codec, r, c)
            total += r * c
            k0 += nk
            r0 += r
    return total


def _encode_matches_oracle(b, Ws):
    """Alg. 1 l.3-5 of the oracle on the INPUT weights with the GPU's scales reproduces the GPU's
    table, offsets and payload byte for byte."""
    _, off, table, _, scales = _host_block(b)
    S, r0 = [], 0
    for (r, _) in b.shapes:
        S.append(scales[r0:r0 + r])
        r0 += r
    ref = o.quantize_encode(Ws, scales=S, cs=b.chunk_symbols, codec=b.codec, chunk_mode=b.chunk_mode)
    assert np.array_equal(off, np.asarray(ref.chunk_off, dtype=np.uint32))
    assert b.payload_bytes == len(ref.payload)
    assert b.payload[:b.payload_bytes].cpu().numpy().tobytes() == ref.payload


def test_config2_llama_1b_every_symbol_and_sampled_encode():
    """BASELINE config 2 (Llama-3.2-1B shapes, 16 blocks, 0.97 G parameters), the bench's encoding
    (R18 pair codec, R17 interleaved chunks): λ calibrated for 2 bits on the GPU, Alg. 1 for every block, one decode launch; every
    symbol against the oracle's decoder, block 7's encode against the oracle's."""
    dev = torch.device("cuda")
    calib = eqsynth.block_weights("llama-3.2-1b", 0, device=dev)
    lam, _ = eq.calibrate_lambda(calib, 2.0, row_stride=16, codec=eq.EQ_CODEC_PAIR_G,
                                 chunk_mode=eq.EQ_CHUNK_INTERLEAVED)
    del calib
    blocks, kept = [], None
    for lid in range(16):
        Ws = eqsynth.block_weights("llama-3.2-1b", lid, device=dev)
        blocks.append(eq.quantize_encode(Ws, lam=lam, codec=eq.EQ_CODEC_PAIR_G, chunk_mode=eq.EQ_CHUNK_INTERLEAVED))
        if lid == 7:
            kept = [W.cpu() for W in Ws]
        del Ws
    n = _decode_all_vs_oracle(blocks)
    assert n == 16 * 60817408
    _encode_matches_oracle(blocks[7], kept)
    bits = 8 * sum(b.compressed_bytes() for b in blocks) / n
    assert abs(bits - 2.0) < 0.05


def test_config5_llama_70b_block_every_symbol_and_encode():
    """BASELINE config 5 (Llama-3-70B shapes; the per-rank parity of §8(d) is on sampled
    blocks): one whole 70B block (856 M parameters) in the bench's encoding — every symbol
    of its decode against the oracle's decoder, and its encode against the oracle's."""
    dev = torch.device("cuda")
    Ws = eqsynth.block_weights("llama-3-70b", 3, device=dev)
    b = eq.quantize_encode(Ws, lam=LAM, codec=eq.EQ_CODEC_PAIR_G, chunk_mode=eq.EQ_CHUNK_INTERLEAVED)
    Wc = [W.cpu() for W in Ws]
    del Ws
    torch.cuda.empty_cache()
    assert _decode_all_vs_oracle([b]) == 855638016
    _encode_matches_oracle(b, Wc)
