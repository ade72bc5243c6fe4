"""GPU parity: every §8(a) row through the C-ABI against the oracle on the same seeded inputs.

Bit-exact for symbols, streams, offsets, tables, codes, dequantised bf16 (given identical
scales); the scale search is compared as the north_star states (objective within 1e-6
relative; identical scale except documented near-ties, which must be optimal under the
oracle's objective table).
"""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq

pytestmark = pytest.mark.gpu

DEV = "cuda"


def u16(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def to_bf16(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(DEV)


def table_u16(blk: o.OracleBlock) -> np.ndarray:
    """The block's table buffer in the device layout of include/entquant.h: the 256 single
    frequencies, plus for EQ_CODEC_PAIR the pair table, escape, K and the rank codes."""
    if blk.codec not in o.PAIR_CODECS:
        return np.ascontiguousarray(blk.freq, dtype=np.uint16)
    t = np.zeros(512, dtype=np.uint16)
    t[:256] = blk.freq
    t[256:481] = blk.pair.pf
    t[481] = blk.pair.fesc
    t[482] = blk.pair.K
    t.view(np.uint8)[968:984] = blk.pair.rank_code
    return t


def oracle_block_to_gpu(blk: o.OracleBlock) -> eq.Block:
    cap = (len(blk.payload) + eq.EQ_PAYLOAD_SLACK + 255) // 256 * 256
    payload = torch.zeros(cap, dtype=torch.uint8)
    payload[:len(blk.payload)] = torch.frombuffer(bytearray(blk.payload), dtype=torch.uint8) if blk.payload else payload[:0]
    off = torch.from_numpy(blk.chunk_off.astype(np.int64).astype(np.int32))
    freq = torch.from_numpy(table_u16(blk).view(np.int16).copy())
    scales = to_bf16(np.concatenate(blk.scales))
    return eq.Block(payload.to(DEV), len(blk.payload), off.to(DEV), freq.to(DEV), scales, list(blk.layer_shapes),
                    blk.chunk_symbols, format=blk.fmt, codec=blk.codec, chunk_mode=blk.chunk_mode)


RAGGED = [(37, 53), (1, 1), (64, 64), (5, 4097), (16, 4096)]


def small_layers(seed=1, shapes=RAGGED, dist="t4"):
    return [eqsynth.weights(r, c, seed=seed, layer=0, matrix=m, dist=dist) for m, (r, c) in enumerate(shapes)]


# ------------------------------------------------------------------ a7/a8 decode
@pytest.mark.parametrize("cs", [4096, 1000, 64, 1])
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16])
def test_decode_oracle_streams(cs, out):
    layers = small_layers()
    scales = [o.absmax_scales(W) for W in layers]
    scales[2] = (scales[2].astype(np.int32) + 1700).astype(np.uint16)       # ~2-bit regime rows
    blk = o.quantize_encode(layers, scales=scales, cs=cs)
    views = eq.decode_dequant([oracle_block_to_gpu(blk)], out)[0]
    a = 0
    for (r, c), v, S in zip(blk.layer_shapes, views, blk.scales):
        codes = blk.codes[a:a + r * c].reshape(r, c)
        a += r * c
        if out == eq.EQ_OUT_FP8:
            assert (v.view(torch.uint8).cpu().numpy() == codes).all()
        else:
            assert (u16(v) == o.dequant(codes, S)).all()


def test_decode_many_blocks_one_launch():
    blocks, refs = [], []
    for b in range(5):
        layers = small_layers(seed=10 + b, shapes=[(32, 256), (7, 96), (48, 512)])
        scales = [(o.absmax_scales(W).astype(np.int32) + 128 * (6 + b)).astype(np.uint16) for W in layers]
        ob = o.quantize_encode(layers, scales=scales, cs=512)
        blocks.append(oracle_block_to_gpu(ob))
        refs.append(o.decode_dequant(ob))
    views = eq.decode_dequant(blocks, eq.EQ_OUT_BF16)
    for vb, rb in zip(views, refs):
        for v, r in zip(vb, rb):
            assert (u16(v) == r).all()


def test_decode_detects_corruption_and_truncation():
    layers = small_layers(shapes=[(64, 512)])
    blk = o.quantize_encode(layers, lam=None, cs=512)
    g = oracle_block_to_gpu(blk)
    d = eq.Decoder([g], eq.EQ_OUT_FP8)
    d()
    d.check()
    # flip a byte in the middle of chunk 3
    a, b = int(blk.chunk_off[3]), int(blk.chunk_off[4])
    g.payload[(a + b) // 2] ^= 0x5A
    d.err.zero_()
    d()
    with pytest.raises(eq.EqError) as ei:
        d.check()
    assert ei.value.status == eq.EQ_ERR_CORRUPT
    g.payload[(a + b) // 2] ^= 0x5A
    # offsets beyond the payload -> truncated
    g.chunk_off[-1] = blk.chunk_off[-1] + 1000
    d.err.zero_()
    d()
    with pytest.raises(eq.EqError) as ei:
        d.check()
    assert ei.value.status == eq.EQ_ERR_TRUNCATED
    # undersized arena -> buffer (synchronous)
    with pytest.raises(eq.EqError) as ei:
        eq.Decoder([g], eq.EQ_OUT_BF16, arena=torch.empty(100, dtype=torch.uint8, device=DEV))
    assert ei.value.status == eq.EQ_ERR_BUFFER


# ------------------------------------------------------------------ a1 / a3 / a4
def test_absmax_vs_oracle():
    for W in small_layers() + [eqsynth.weights(300, 700, seed=4, dist="mix")]:
        Wd = W.to(DEV)
        Wd[0].zero_() if W.shape[0] > 3 else None
        assert (u16(eq.absmax(Wd)) == o.absmax_scales(Wd.cpu())).all()


def test_quantize_hist_vs_oracle():
    for i, W in enumerate(small_layers() + [eqsynth.weights(256, 1024, seed=5, dist="t3", outliers=3)]):
        S = o.absmax_scales(W)
        S = (S.astype(np.int32) + 64 * (i % 5) * 20).astype(np.uint16)
        codes, hist = eq.quantize_hist(W.to(DEV), to_bf16(S))
        ref = o.quantize(W, S)
        assert (codes.cpu().numpy() == ref).all()
        assert (hist.cpu().numpy().astype(np.uint64) == o.histogram(ref)).all()


def test_quantize_exhaustive_bf16_patterns():
    """All finite bf16 W patterns under a few scales — the tie rule and the clamp."""
    bits = np.arange(0x10000, dtype=np.uint32).astype(np.uint16)
    fin = ((bits & 0x7F80) != 0x7F80)
    W = bits[fin][: (fin.sum() // 256) * 256].reshape(256, -1)
    for s in [0x3F80, 0x3C00, 0x4040, 0x3700, 0x4430]:
        S = np.full(256, s, dtype=np.uint16)
        codes, _ = eq.quantize_hist(to_bf16(W), to_bf16(S))
        assert (codes.cpu().numpy() == o.quantize(W, S)).all(), hex(s)


# ------------------------------------------------------------------ a5
@pytest.mark.parametrize("kind", ["skewed", "uniform", "subset130", "subset248", "single", "weights"])
def test_build_table_vs_oracle(kind):
    if kind == "weights":
        W = eqsynth.weights(128, 512, seed=3)
        h = o.histogram(o.quantize(W, (o.absmax_scales(W).astype(np.int32) + 1800).astype(np.uint16)))
    else:
        h = o.histogram(eqsynth.random_codes_stream(77777, 5, kind))
    freq, err = eq.build_table(torch.from_numpy(h.astype(np.int64)).to(DEV))
    eq.check(err)
    assert (freq.cpu().numpy().view(np.uint16) == o.normalize(h)).all()
    _, err = eq.build_table(torch.zeros(256, dtype=torch.int64, device=DEV))
    with pytest.raises(eq.EqError):
        eq.check(err)


# ------------------------------------------------------------------ a6
@pytest.mark.parametrize("cs", [4096, 333])
def test_rans_encode_byte_identical(cs):
    layers = small_layers()
    scales = [(o.absmax_scales(W).astype(np.int32) + 1500).astype(np.uint16) for W in layers]
    blk = o.quantize_encode(layers, scales=scales, cs=cs)
    g = eq.rans_encode(torch.from_numpy(blk.codes).to(DEV), blk.layer_shapes,
                       torch.from_numpy(blk.freq.view(np.int16).copy()).to(DEV), chunk_symbols=cs, codec=eq.EQ_CODEC_BYTE)
    assert g.payload_bytes == len(blk.payload)
    assert (g.chunk_off.cpu().numpy().astype(np.uint32) == blk.chunk_off).all()
    assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == blk.payload


# ------------------------------------------------------------------ a2
def check_search_rows(W, lam, S_gpu, obj_gpu, rows, oct_lo=-1, oct_hi=20):
    """GPU choice == oracle choice, or a documented near-tie: the GPU's scale must be
    optimal under the oracle's objective table to 1e-9 relative."""
    near_ties = 0
    for r in rows:
        first, f = o.row_objectives(W, r, lam, oct_lo, oct_hi)
        k_or = int(np.argmin(f))
        k_gpu = int(S_gpu[r]) - first
        assert 0 <= k_gpu < f.size
        if k_gpu != k_or:
            near_ties += 1
            assert f[k_gpu] <= f[k_or] * (1 + 1e-9), (r, k_gpu, k_or)
        assert obj_gpu[r] == pytest.approx(f[k_or], rel=1e-6)
    return near_ties


@pytest.mark.parametrize("lam", [0.0, 60.0, 250.0])
def test_search_vs_oracle(lam):
    W = eqsynth.weights(24, 384, seed=6)
    W[3].zero_()
    sc, ob = eq.search_scales(W.to(DEV), [lam], with_obj=True)
    S, obj = u16(sc[0]), ob[0].cpu().numpy()
    assert S[3] == 0x3F80
    rows = [r for r in range(24) if r != 3]
    assert check_search_rows(W, lam, S, obj, rows) <= 1
    S_or, f_or = o.search(W, lam)
    assert np.mean(S == S_or) > 0.95


@pytest.mark.parametrize("lam", [0.0, 100.0])
def test_search_exact_midpoint_ties(lam):
    """Rows whose quotients w/s are EXACT E4M3 rounding midpoints (ties, §8c.3: RNE takes the
    even code) at the single candidate s = s0 = 2^k (bracket [0, 0]): the GPU objective of that
    candidate — the division-free search decides ties by two perturbed products — equals the
    oracle's exact-quotient objective.  A tie rounded away from even changes R = Σ|v|."""
    vals = sorted({o.e4m3_value(c) for c in range(0x7F)})            # 0 .. 448
    mids = [(a + b) / 2 for a, b in zip(vals[:-1], vals[1:])]         # 126 midpoints, exact in bf16
    rows = []
    for k in (-6, -2, 0, 3):
        r = [448.0] + mids + [-m for m in mids] + [3.0, -0.5, 100.0]
        rows.append(np.array(r[:256] + [0.0] * (256 - len(r)), dtype=np.float64) * 2.0 ** k)
    W = torch.from_numpy(np.stack(rows)).to(torch.bfloat16)
    assert torch.equal(W.double(), torch.from_numpy(np.stack(rows)))  # exact in bf16
    _, ob = eq.search_scales(W.to(DEV), [lam], oct_lo=0, oct_hi=0, with_obj=True)
    for r in range(4):
        first, f = o.row_objectives(W, r, lam, 0, 0)
        assert f.size == 1
        assert float(ob[0, r]) == pytest.approx(f[0], rel=1e-12), r


def test_search_multi_lambda_and_row_subset():
    W = eqsynth.weights(40, 256, seed=7, dist="mix")
    lams = [0.0, 10.0, 100.0, 400.0]
    full = eq.search_scales(W.to(DEV), lams)
    rows = torch.tensor([1, 5, 17, 39], dtype=torch.int32)
    sub = eq.search_scales(W.to(DEV), lams, rows=rows)
    for k, lam in enumerate(lams):
        single = eq.search_scales(W.to(DEV), [lam])[0]
        assert torch.equal(full[k].view(torch.int16), single.view(torch.int16))
        assert torch.equal(sub[k, rows.long()].view(torch.int16), full[k, rows.long()].view(torch.int16))


# ------------------------------------------------------------------ Alg. 1 end to end (config 1)
def test_config1_full_pipeline_vs_oracle():
    """BASELINE config 1: 256x256 Student-t matrix, per-row scales, E4M3 + rANS in 4096-symbol
    chunks; GPU search+quantise+table+encode vs the full oracle pipeline."""
    W = eqsynth.weights(256, 256, seed=0)
    lam = 150.0
    g = eq.quantize_encode([W.to(DEV)], lam=lam, codec=eq.EQ_CODEC_BYTE)
    S_gpu = u16(g.scales)
    S_or, f_or = o.search(W, lam)
    _, ob = eq.search_scales(W.to(DEV), [lam], with_obj=True)
    diff = np.nonzero(S_gpu != S_or)[0]
    check_search_rows(W, lam, S_gpu, ob[0].cpu().numpy(), list(diff) + [0, 1, 2])
    # with the oracle's own scales the GPU stream is the oracle's bit for bit
    g2 = eq.quantize_encode([W.to(DEV)], scales=to_bf16(S_or), codec=eq.EQ_CODEC_BYTE)
    ref2 = o.quantize_encode([W], scales=[S_or])
    assert (g2.freq.cpu().numpy().view(np.uint16) == ref2.freq).all()
    assert (g2.chunk_off.cpu().numpy().astype(np.uint32) == ref2.chunk_off).all()
    if diff.size == 0:   # no near-tie rows: the searched block is the oracle's block
        assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == ref2.payload
    assert g2.payload[:g2.payload_bytes].cpu().numpy().tobytes() == ref2.payload
    # decode + dequant round trip
    v = eq.decode_dequant([g2], eq.EQ_OUT_BF16)[0][0]
    assert (u16(v) == o.decode_dequant(ref2)[0]).all()
    H = o.entropy(ref2.hist)
    assert g2.payload_bytes + 4 * (g2.n_chunks + 1) <= 1.02 * W.numel() * H / 8


def test_quantize_encode_absmax_and_ragged():
    layers = small_layers(seed=3)
    for cs in [4096, 100]:
        g = eq.quantize_encode([W.to(DEV) for W in layers], scale_mode=eq.EQ_SCALES_ABSMAX, chunk_symbols=cs, codec=eq.EQ_CODEC_BYTE)
        ref = o.quantize_encode(layers, lam=None, cs=cs)
        assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == ref.payload
        for v, r in zip(eq.decode_dequant([g], eq.EQ_OUT_BF16)[0], o.decode_dequant(ref)):
            assert (u16(v) == r).all()


def test_host_buffer_e2e_decode():
    layers = small_layers(seed=8, shapes=[(64, 256), (32, 512)])
    g = eq.quantize_encode([W.to(DEV) for W in layers], lam=80.0, codec=eq.EQ_CODEC_BYTE)
    hb = eq.HostBlocks([g], eq.EQ_OUT_BF16)
    arena = hb.decode()
    dev = eq.Decoder([g], eq.EQ_OUT_BF16)
    dev()
    dev.check()
    assert torch.equal(arena[:dev.total], dev.arena[:dev.total].cpu())


def test_calibrate_lambda_reaches_target():
    layers = [eqsynth.weights(r, c, seed=2, layer=0, matrix=m) for m, (r, c) in enumerate([(128, 512), (256, 512)])]
    dl = [W.to(DEV) for W in layers]
    lam, est = eq.calibrate_lambda(dl, 2.5, row_stride=2, codec=eq.EQ_CODEC_BYTE)
    assert abs(est - 2.5) < 0.1
    g = eq.quantize_encode(dl, lam=lam, codec=eq.EQ_CODEC_BYTE)
    assert abs(g.effective_bits() - 2.5) < 0.35
    with pytest.raises(eq.EqError) as ei:
        eq.calibrate_lambda(dl, 9.5, row_stride=4, codec=eq.EQ_CODEC_BYTE)
    assert ei.value.status == eq.EQ_ERR_UNREACHABLE_TARGET


def test_calibrate_lambda_full_block_within_005_bits():
    """λ for a target rate within ±0.05 effective bits, at the bench's scale (one
    Llama-3-8B-shaped block, pair codec, row chunks of 4096): calibrate on sampled rows, then
    encode the whole block."""
    Ws = eqsynth.block_weights("llama-3-8b", 3, device=DEV)
    for target in (2.0, 3.0):
        lam, est = eq.calibrate_lambda(Ws, target, row_stride=16, codec=eq.EQ_CODEC_PAIR, chunk_mode=eq.EQ_CHUNK_ROW)
        assert abs(est - target) < 0.05, (target, est)
        g = eq.quantize_encode(Ws, lam=lam, codec=eq.EQ_CODEC_PAIR, chunk_mode=eq.EQ_CHUNK_ROW)
        assert abs(g.effective_bits() - target) < 0.05, (target, g.effective_bits())


ENCODINGS = [(o.CODEC_BYTE, o.CHUNK_LAYER), (o.CODEC_PAIR, o.CHUNK_LAYER), (o.CODEC_PAIR_G, o.CHUNK_INTERLEAVED),
             (o.CODEC_PAIR_G, o.CHUNK_LAYER)]
ENC_IDS = ["byte", "pair", "pairg-il", "pairg"]


@pytest.mark.parametrize("codec,mode", ENCODINGS, ids=ENC_IDS)
def test_dequant_all_codes_all_scale_ranges(codec, mode):
    """Every finite E4M3 code × row scales across the bf16 range (f16-exact scales take the
    FHFMA path, the rest the FMUL path; subnormal bf16 products included; the R18 bf16 path
    multiplies bf16 value pairs by the bf16 scale), decoded through the C-ABI and compared with
    the oracle's exact dequantiser."""
    codes = np.array([c for c in range(256) if (c & 0x7F) != 0x7F and c != 0x80], dtype=np.uint8)   # 253
    row = np.concatenate([codes, codes[:3]])                                                       # 256 cols
    rng = np.random.default_rng(11)
    s_bits = np.concatenate([
        rng.integers(0x0080, 0x3800, 40),     # below the f16 normal range (FMUL path), incl. tiny
        rng.integers(0x3880, 0x4780, 40),     # f16-exact range (FHFMA path)
        rng.integers(0x4780, 0x7B00, 40),     # above f16 max (FMUL path)
        [0x0001, 0x0005, 0x3880, 0x387F, 0x477F, 0x4780, 0x3F80],
    ]).astype(np.uint16)
    M = s_bits.size
    C = np.tile(row, (M, 1))
    blk = o.encode_codes([C], [(M, 256)], [s_bits], cs=512, codec=codec, chunk_mode=mode)
    v = eq.decode_dequant([oracle_block_to_gpu(blk)], eq.EQ_OUT_BF16)[0][0]
    assert (u16(v) == o.dequant(C, s_bits)).all()


# ------------------------------------------------------------------ NEXT row 4: Int8 + exclusion
I8 = eq.EQ_FMT_INT8


def test_int8_absmax_quantize_exhaustive():
    bits = np.arange(0x10000, dtype=np.uint32).astype(np.uint16)
    fin = ((bits & 0x7F80) != 0x7F80)
    W = bits[fin][: (fin.sum() // 256) * 256].reshape(256, -1)
    for s in [0x3F80, 0x3C00, 0x4040, 0x3700, 0x4430]:
        S = np.full(256, s, dtype=np.uint16)
        codes, hist = eq.quantize_hist(to_bf16(W), to_bf16(S), format=I8)
        ref = o.quantize(W, S, o.FMT_INT8)
        assert (codes.cpu().numpy() == ref).all(), hex(s)
        assert (hist.cpu().numpy().astype(np.uint64) == o.histogram(ref)).all()
    for Wt in small_layers():
        assert (u16(eq.absmax(Wt.to(DEV), format=I8)) == o.absmax_scales(Wt, o.FMT_INT8)).all()


@pytest.mark.parametrize("lam", [0.0, 120.0])
def test_int8_search_vs_oracle(lam):
    W = eqsynth.weights(16, 320, seed=13)
    sc, ob = eq.search_scales(W.to(DEV), [lam], with_obj=True, format=I8)
    S = u16(sc[0])
    obj = ob[0].cpu().numpy()
    near = 0
    for r in range(16):
        first, f = o.row_objectives(W, r, lam, fmt=o.FMT_INT8)
        k = int(S[r]) - first
        if k != int(np.argmin(f)):
            near += 1
            assert f[k] <= f.min() * (1 + 1e-9)
        assert obj[r] == pytest.approx(f.min(), rel=1e-6)
    assert near <= 1


@pytest.mark.parametrize("codec,mode", ENCODINGS, ids=ENC_IDS)
@pytest.mark.parametrize("out", [eq.EQ_OUT_FP8, eq.EQ_OUT_BF16])
def test_int8_decode_oracle_streams(out, codec, mode):
    shapes = RAGGED if mode == o.CHUNK_LAYER else [(37, 64), (1, 16), (64, 64), (5, 4096), (16, 4096)]
    layers = small_layers(seed=21, shapes=shapes)
    scales = [(o.absmax_scales(W, o.FMT_INT8).astype(np.int32) + 128 * 5).astype(np.uint16) for W in layers]
    blk = o.quantize_encode(layers, scales=scales, cs=512, fmt=o.FMT_INT8, codec=codec, chunk_mode=mode)
    views = eq.decode_dequant([oracle_block_to_gpu(blk)], out)[0]
    a = 0
    for (r, c), v, S in zip(blk.layer_shapes, views, blk.scales):
        codes = blk.codes[a:a + r * c].reshape(r, c)
        a += r * c
        if out == eq.EQ_OUT_FP8:
            assert (v.view(torch.uint8).cpu().numpy() == codes).all()
        else:
            assert (u16(v) == o.dequant(codes, S, o.FMT_INT8)).all()


@pytest.mark.parametrize("fmt", [eq.EQ_FMT_E4M3, eq.EQ_FMT_INT8])
def test_quantize_encode_format_and_exclusion(fmt):
    layers = [eqsynth.weights(r, c, seed=22, layer=1, matrix=m) for m, (r, c) in enumerate([(48, 256), (32, 512), (8, 4096)])]
    lam = 150.0
    g = eq.quantize_encode([W.to(DEV) for W in layers], lam=lam, format=fmt, exclude=(2,), codec=eq.EQ_CODEC_BYTE)
    S_gpu = u16(g.scales)
    assert (S_gpu[80:88] == o.absmax_scales(layers[2], fmt)).all()              # excluded layer: λ = 0
    S_or = [o.search(W, lam, fmt=fmt)[0] for W in layers[:2]] + [o.absmax_scales(layers[2], fmt)]
    sc = to_bf16(np.concatenate(S_or))
    g2 = eq.quantize_encode([W.to(DEV) for W in layers], scales=sc, format=fmt, codec=eq.EQ_CODEC_BYTE)
    ref = o.quantize_encode(layers, scales=S_or, fmt=fmt)
    assert g2.payload[:g2.payload_bytes].cpu().numpy().tobytes() == ref.payload
    for v, r in zip(eq.decode_dequant([g2], eq.EQ_OUT_BF16)[0], o.decode_dequant(ref)):
        assert (u16(v) == r).all()
    if (S_gpu == np.concatenate(S_or)).all():
        assert g.payload[:g.payload_bytes].cpu().numpy().tobytes() == ref.payload
