"""The CRC verify mode on the GPU: eq_crc32 against the oracle's
CRC-32 (zlib) on every length class and alignment, the block CRC recorded at encode time against
the oracle's codes, and the verify path over a decode (incl. a full Llama-3-8B block)."""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq
from test_gpu_parity import DEV, to_bf16

pytestmark = pytest.mark.gpu


def test_crc32_check_value_on_gpu():
    t = torch.frombuffer(bytearray(b"123456789"), dtype=torch.uint8).to(DEV)
    assert eq.crc32(t) == 0xCBF43926
    assert eq.crc32(torch.zeros(0, dtype=torch.uint8, device=DEV)) == 0


@pytest.mark.parametrize("n", [1, 3, 15, 16, 17, 4095, 4096, 4097, 8192 + 5, (1 << 20) + 123, 4096 * 1100 + 7,
                               4096 * 5000])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_crc32_matches_oracle(n, offset):
    """Pieces of 4 KB (ragged last piece), runs of pieces folded per thread (ragged last run),
    16-byte vector loads and unaligned byte starts."""
    rng = np.random.default_rng(n + offset)
    host = rng.integers(0, 256, n + offset, dtype=np.uint8)
    dev = torch.from_numpy(host).to(DEV)
    assert eq.crc32(dev[offset:]) == o.crc32(host[offset:]), (n, offset)


@pytest.mark.parametrize("codec,mode", [(eq.EQ_CODEC_PAIR_G, eq.EQ_CHUNK_INTERLEAVED), (eq.EQ_CODEC_WORD, eq.EQ_CHUNK_LAYER)])
def test_block_crc_recorded_at_encode_and_verified(codec, mode):
    shapes = [(64, 4096), (24, 704), (48, 1024)]
    layers = [eqsynth.weights(r, c, seed=31, layer=0, matrix=m) for m, (r, c) in enumerate(shapes)]
    S = [(o.absmax_scales(W).astype(np.int32) + 128 * 12).astype(np.uint16) for W in layers]
    g = eq.quantize_encode([W.to(DEV) for W in layers], scales=to_bf16(np.concatenate(S)), codec=codec,
                           chunk_mode=mode, chunk_symbols=256, crc=True)
    ref = o.quantize_encode(layers, scales=S, cs=256, codec=codec, chunk_mode=mode)
    assert g.crc == o.crc32(ref.codes)                   # the codes in layer order
    assert eq.verify_crc([g]) == [True]
    bad = eq.Block(g.payload.clone(), g.payload_bytes, g.chunk_off, g.freq, g.scales, g.shapes, g.chunk_symbols,
                   g.meta, g.format, g.codec, g.chunk_mode, g.crc ^ 1)
    assert eq.verify_crc([bad]) == [False]             # a recorded CRC that does not match


def test_block_crc_full_llama_block():
    Ws = eqsynth.block_weights("llama-3-8b", 0, device=DEV)
    g = eq.quantize_encode(Ws, lam=230.2, crc=True, chunk_mode=eq.EQ_CHUNK_INTERLEAVED)
    dec = eq.Decoder([g], eq.EQ_OUT_FP8)
    dec()
    dec.check()
    codes = torch.cat([v.reshape(-1).view(torch.uint8) for v in dec.views()[0]]).cpu().numpy()
    assert o.crc32(codes) == g.crc                      # 218 M codes, 53 K pieces
    assert eq.verify_crc([g]) == [True]
