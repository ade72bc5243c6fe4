"""GPU parity for the pair codec (EQ_CODEC_PAIR, reading R15): decode of
oracle-encoded streams (symbols and bf16 bit-exact), incl. escapes, odd chunk lengths and
ragged layers; GPU encode byte-identical to the oracle."""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq
from test_gpu_parity import DEV, oracle_block_to_gpu, small_layers, to_bf16, u16

pytestmark = pytest.mark.gpu
PAIR = o.CODEC_PAIR


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
@pytest.mark.parametrize("cs", [4096, 1000, 64, 7, 1])
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16])
def test_pair_decode_oracle_streams(cs, out, pc):
    layers = small_layers()
    scales = [o.absmax_scales(W) for W in layers]
    scales[2] = (scales[2].astype(np.int32) + 1700).astype(np.uint16)
    scales[4] = (scales[4].astype(np.int32) + 2000).astype(np.uint16)
    blk = o.quantize_encode(layers, scales=scales, cs=cs, codec=pc)
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
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16], ids=["fp8", "bf16"])
@pytest.mark.parametrize("kind", ["uniform", "subset2", "single", "skewed", "subset40"])
def test_pair_decode_extreme_streams(kind, out, pc):
    """Escape-heavy (uniform bytes: 15 of 256 codes ranked), single-code and two-code tables.
    The single-code table's (0,0) pair has f > 2048, so it also runs the decoder's wide LUT
    entries (the narrow 2·id layout needs every kept pair at f ≤ 2048)."""
    s = eqsynth.random_codes_stream(64 * 4096, 3, kind)
    s = np.where((s & 0x7F) == 0x7F, s ^ 1, s).astype(np.uint8)       # no NaN codes (never produced, R1)
    S = (np.arange(64, dtype=np.uint16) * 37 + 0x3C00).astype(np.uint16)
    blk = o.encode_codes([s.reshape(64, 4096)], [(64, 4096)], [S], 4096, codec=pc)
    v = eq.decode_dequant([oracle_block_to_gpu(blk)], out)[0][0]
    if out == eq.EQ_OUT_FP8:
        assert (v.view(torch.uint8).cpu().numpy().reshape(-1) == s).all()
    else:
        assert (u16(v) == o.dequant(s.reshape(64, 4096), S)).all()


def _pair_hists():
    """Histograms for the pair-table kernel: the hand-derived golden cases, escape-heavy and
    single-code streams, heavy heads over many count-1 codes (D < 0), random Pareto counts,
    and a 2-bit weight matrix."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "normalize_worked.json")))
    from test_oracle_codec import _expand, hist_of
    hs = [hist_of(_expand(c["counts"])) for c in g["pair_cases"] + g["cases"]]
    for kind in ["uniform", "subset2", "single", "skewed", "subset40", "subset130", "subset248"]:
        hs.append(o.histogram(eqsynth.random_codes_stream(50000, 7, kind)))
    rng = np.random.default_rng(5)
    for t in range(40):
        k = int(rng.integers(1, 257))
        h = np.zeros(256, np.uint64)
        idx = rng.permutation(256)[:k]
        h[idx] = (rng.pareto(0.3 + rng.uniform(0, 3), k) * rng.choice([1, 10, 1000, 1e6])).astype(np.uint64) + 1
        if t % 4 == 0:
            h[idx[: k // 2]] = 1
        hs.append(h)
    W = eqsynth.weights(256, 4096, seed=6)
    hs.append(o.histogram(o.quantize(W, (o.absmax_scales(W).astype(np.int32) + 1900).astype(np.uint16))))
    big = np.zeros(256, np.uint64)                   # block-sized counts (8B down_proj scale)
    big[[0, 1, 255, 8, 136]] = [91_000_000, 40_000_000, 39_000_000, 3_000_000, 1]
    hs.append(big)
    return hs


def test_pair_table_kernel_vs_oracle():
    """k_build_pair_table (device, R15 written as rank counting + water-filling) equals the
    oracle's pair_table on every histogram, entry for entry, incl. K, escape and rank codes."""
    for i, h in enumerate(_pair_hists()):
        tab, err = eq.build_pair_table(torch.from_numpy(h.astype(np.int64)).to(DEV))
        eq.check(err)
        pt = o.pair_table(h)
        want = np.zeros(512, np.uint16)
        want[:256] = o.normalize(h)
        want[256:481] = pt.pf
        want[481] = pt.fesc
        want[482] = pt.K
        want.view(np.uint8)[968:984] = pt.rank_code
        got = tab.cpu().numpy().view(np.uint16)
        assert (got == want).all(), (i, np.nonzero(got != want))
    _, err = eq.build_pair_table(torch.zeros(256, dtype=torch.int64, device=DEV))
    with pytest.raises(eq.EqError):
        eq.check(err)


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
@pytest.mark.parametrize("cs", [4096, 333, 1])
def test_pair_quantize_encode_byte_identical(cs, pc):
    """Alg. 1 on the GPU with the pair codec, given the oracle's scales: the table buffer
    (single + pair tables, both built by device kernels) and the stream are the oracle's."""
    from test_gpu_parity import table_u16
    layers = small_layers(seed=5)
    S = [(o.absmax_scales(W).astype(np.int32) + 1500).astype(np.uint16) for W in layers]
    g = eq.quantize_encode([W.to(DEV) for W in layers], scales=to_bf16(np.concatenate(S)), chunk_symbols=cs,
                           codec=pc)
    ref = o.quantize_encode(layers, scales=S, cs=cs, codec=pc)
    assert (g.freq.cpu().numpy().view(np.uint16) == table_u16(ref)).all()
    assert g.payload_bytes == len(ref.payload)
    assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == ref.payload
    for v, r in zip(eq.decode_dequant([g], eq.EQ_OUT_BF16)[0], o.decode_dequant(ref)):
        assert (u16(v) == r).all()


def test_pair_rate_at_two_bits_gpu():
    W = eqsynth.weights(512, 4096, seed=6)
    gp = eq.quantize_encode([W.to(DEV)], lam=230.0, codec=eq.EQ_CODEC_PAIR)
    codes, hist = eq.quantize_hist(W.to(DEV), gp.scales)
    H = o.entropy(hist.cpu().numpy().astype(np.uint64))
    assert gp.payload_bytes + 4 * (gp.n_chunks + 1) <= 1.02 * W.numel() * H / 8


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
def test_pair_host_buffer_e2e_decode(pc):
    layers = small_layers(seed=8, shapes=[(64, 256), (32, 512)])
    g = eq.quantize_encode([W.to(DEV) for W in layers], lam=80.0, codec=pc)
    hb = eq.HostBlocks([g], eq.EQ_OUT_BF16)
    arena = hb.decode()
    dev = eq.Decoder([g], eq.EQ_OUT_BF16)
    dev()
    dev.check()
    assert torch.equal(arena[:dev.total], dev.arena[:dev.total].cpu())


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
def test_pair_runaway_stream_is_reported(pc):
    """A chunk whose state is forced to 1 (every step then escapes or renormalises) runs past
    its end: reported as CORRUPT, never read beyond the payload slack (see memcheck runs)."""
    Ws = [eqsynth.weights(128, 4096, seed=12)]
    blk = o.quantize_encode(Ws, scales=[(o.absmax_scales(Ws[0]).astype(np.int32) + 1700).astype(np.uint16)],
                            cs=2048, codec=pc)
    g = oracle_block_to_gpu(blk)
    a = int(blk.chunk_off[blk.n_chunks - 1])
    g.payload[a:a + 4] = torch.tensor([1, 0, 0, 0], dtype=torch.uint8, device=DEV)
    d = eq.Decoder([g], eq.EQ_OUT_BF16)
    d()
    with pytest.raises(eq.EqError) as ei:
        d.check()
    assert ei.value.status == eq.EQ_ERR_CORRUPT


@pytest.mark.parametrize("pc", [o.CODEC_PAIR, o.CODEC_PAIR_G], ids=["r15", "r18"])
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16], ids=["fp8", "bf16"])
def test_pair_decode_many_tiny_chunks(out, pc):
    """204,800 chunks of 16 symbols in one launch (800 CTAs: a second, thin round on 148 SMs at
    5 CTAs/SM; every chunk is one fast group): the decoded symbols equal the oracle's stream."""
    rows, cols, cs = 800, 4096, 16
    s = eqsynth.random_codes_stream(rows * cols, 5, "skewed")
    s = np.where((s & 0x7F) == 0x7F, s ^ 1, s).astype(np.uint8)
    S = (np.arange(rows, dtype=np.uint16) % 61 + 0x3B80).astype(np.uint16)
    blk = o.encode_codes([s.reshape(rows, cols)], [(rows, cols)], [S], cs, codec=pc)
    assert blk.n_chunks == rows * cols // cs
    v = eq.decode_dequant([oracle_block_to_gpu(blk)], out)[0][0]
    if out == eq.EQ_OUT_FP8:
        assert (v.view(torch.uint8).cpu().numpy().reshape(-1) == s).all()
    else:
        assert (u16(v) == o.dequant(s.reshape(rows, cols), S)).all()


def test_gpu_pair_codec_reproduces_hand_derived_streams():
    """The device path against the hand-derived pair-codec chunks (tests/golden/
    rans_pair_worked.json, no code involved): k_build_pair_table from the counts, the GPU
    encoder on the symbols -> exactly the golden bytes; the GPU decoder on the golden bytes ->
    the symbols (FP8 output = the codes)."""
    import json, os
    from test_oracle_codec import _expand, hist_of
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rans_pair_worked.json")))
    cases = [(c, eq.EQ_CODEC_PAIR) for c in g["cases"]] + [(c, eq.EQ_CODEC_PAIR_G) for c in g["grouped_cases"]]
    for case, codec in cases:                      # R15 streams, then R18's (grouped escapes)
        h = hist_of(_expand(case["counts"]))
        tab, err = eq.build_pair_table(torch.from_numpy(h.astype(np.int64)).to(DEV))
        eq.check(err)
        sym = np.array(case["symbols"], dtype=np.uint8)
        n = sym.size
        blk = eq.rans_encode(torch.from_numpy(sym).to(DEV), [(1, n)], tab, chunk_symbols=4096, codec=codec)
        assert blk.payload[:blk.payload_bytes].cpu().numpy().tobytes().hex() == case["bytes_hex"], case["name"]
        v = eq.decode_dequant([blk], eq.EQ_OUT_FP8)[0][0]
        assert (v.view(torch.uint8).cpu().numpy().reshape(-1) == sym).all(), case["name"]
