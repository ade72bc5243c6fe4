"""Pins for the Int8 base format (SPEC quantgrid S:26-118) and the per-layer
exclusion flag (super-weight layers coded at λ=0, still entropy coded)."""
import ml_dtypes
import numpy as np
import pytest

import eqsynth
import oracle as o

I8 = o.FMT_INT8


def bf16_bits(x):
    return np.asarray(x, dtype=np.float64).astype(ml_dtypes.bfloat16).view(np.uint16)


def bf16_val(b):
    return np.asarray(b, dtype=np.uint16).view(ml_dtypes.bfloat16).astype(np.float64)


def lib_int8_code(r):
    """numpy reference: clamp to ±127, round half to even (np.rint), two's-complement byte."""
    return np.rint(np.clip(r, -127.0, 127.0)).astype(np.int64).astype(np.int8).view(np.uint8)


def test_int8_grid_spec_examples():
    vals = sorted(o.grid_value(c, I8) for c in range(256) if c != 0x80)
    assert vals == list(range(-127, 128))                      # S:61 "255 entries, −127…127"
    assert o.grid_quantize(-1000.0, I8) == (256 - 127) and o.grid_quantize(1000.0, I8) == 127
    # S:70 row [1,-2,4] -> s = 4/127 (stored bf16);  S:79 codes [32, -64, 127] (half to even)
    W = bf16_bits(np.array([[1.0, -2.0, 4.0]]))
    S = o.absmax_scales(W, I8)
    assert bf16_val(S)[0] == bf16_val(bf16_bits(4.0 / 127.0))
    assert o.quantize(W, S, I8).view(np.int8).tolist() == [[32, -64, 127]]
    assert o.grid_quantize(-63.5, I8) == (256 - 64) and o.grid_quantize(62.5, I8) == 62
    assert o.grid_quantize(-0.3, I8) == 0                      # no −0 / −128 ever


def test_int8_quantize_exhaustive_bf16_vs_numpy():
    w_bits = np.arange(0, 0x10000, dtype=np.uint32).astype(np.uint16)
    w = bf16_val(w_bits)
    fin = np.isfinite(w)
    w_bits, w = w_bits[fin][::5], w[fin][::5]
    ties = 0
    for s in [1.0, 0.0078125, 3.0, 0.02734375, 1.5e-5, 7.0e2]:
        sb = int(bf16_bits(s))
        sv = bf16_val(sb)
        ref = lib_int8_code(w / sv)
        got = o.quantize(w_bits.reshape(1, -1), np.array([sb], np.uint16), I8)[0]
        assert (got == ref).all(), s
        # the f32 quotient rounds identically (the GPU premise)
        assert (lib_int8_code((w.astype(np.float32) / np.float32(sv)).astype(np.float64)) == ref).all()
        r = np.abs(w / sv)
        ties += int(np.sum((r <= 127) & (r == np.floor(r) + 0.5)))
    assert ties > 50


def test_int8_dequant_vs_ml_dtypes():
    rng = np.random.default_rng(3)
    s_bits = np.concatenate([rng.integers(0x0001, 0x7B00, 300), [0x3F80]]).astype(np.uint16)
    codes = np.array([c for c in range(256) if c != 0x80], dtype=np.uint8)
    got = o.dequant(np.tile(codes, (s_bits.size, 1)), s_bits, I8)
    ref = bf16_bits(bf16_val(s_bits)[:, None] * codes.view(np.int8).astype(np.float64)[None, :])
    assert (got == ref).all()


@pytest.mark.parametrize("lam", [0.0, 50.0, 400.0])
def test_int8_search_brute_force(lam):
    W = o._u16(eqsynth.weights(5, 40, seed=12))
    S, fr = o.search(W, lam, -1, 6, fmt=I8)
    Wv = bf16_val(W)
    for i in range(5):
        row = Wv[i]
        s0 = bf16_val(bf16_bits(np.abs(row).max() / 127.0))
        lo, hi = int(bf16_bits(s0 * 0.5)), int(bf16_bits(s0 * 64))
        cands = np.arange(lo, hi + 1, dtype=np.uint16)
        sv = bf16_val(cands)[:, None]
        v = lib_int8_code(row[None, :] / sv).view(np.int8).astype(np.float64)
        f = np.abs(row[None, :] - sv * v).sum(1) / np.abs(Wv).sum() + lam * np.abs(v).sum(1) / Wv.size
        assert S[i] == cands[int(np.argmin(f))]
        assert fr[i] == pytest.approx(f.min(), rel=1e-12)


def test_int8_block_round_trip_and_exclusion():
    layers = [eqsynth.weights(r, c, seed=2, layer=0, matrix=m) for m, (r, c) in enumerate([(32, 128), (16, 256)])]
    blk = o.quantize_encode(layers, lam=200.0, fmt=I8, exclude=(1,))
    assert (blk.scales[1] == o.absmax_scales(layers[1], I8)).all()          # excluded: λ = 0
    assert not (blk.scales[0] == o.absmax_scales(layers[0], I8)).all()
    assert (o.decode_block(blk) == blk.codes).all()
    for W, S, D in zip(layers, blk.scales, o.decode_dequant(blk)):
        assert (D == o.dequant(o.quantize(W, S, I8), S, I8)).all()
    assert 0x80 not in set(blk.codes.tolist())
    # λ=0 Int8 rate is in the 8-bit regime minus entropy gain; excluded layers stay high-rate
    e = o.quantize_encode(layers, lam=None, fmt=I8)
    assert 4.0 < e.effective_bits() < 8.5
