"""Pins for the oracle's metadata and entropy-codec steps (histogram, Ĥ, table
normalisation, rANS, block stream, effective bits).

Expected values: SPEC worked examples (tests/golden/spec_examples.json), hand-derived rANS
streams (tests/golden/rans_worked.json), Shannon's bound, the table cross-entropy bound,
losslessness, chunk independence, and the paper's loose context anchors (≈6.5 bits at λ=0,
P:257; ≫4 unique codes at ~2 bits, Table 1).
"""
import math

import numpy as np
import pytest

import eqsynth
import oracle as o


def hist_of(counts: dict) -> np.ndarray:
    h = np.zeros(256, dtype=np.uint64)
    for k, v in counts.items():
        h[int(k)] = v
    return h


def xent_bits(hist, freq) -> float:
    """Σ c_s·(12 − log2 f_s): ideal coded size of the stream under the 12-bit table."""
    return float(sum(int(c) * (12 - math.log2(int(f))) for c, f in zip(hist, freq) if c))


def emp_entropy_bits(hist) -> float:
    """n·Ĥ computed directly with numpy (Eq. 2)."""
    h = hist[hist > 0].astype(np.float64)
    n = h.sum()
    return float(-(h * np.log2(h / n)).sum())


# ------------------------------------------------------------------ histogram / Ĥ
def test_entropy_examples(golden):
    for ex in golden["spec_examples"]["entropy"]:
        h = hist_of({i: c for i, c in enumerate(ex["counts"])})
        assert o.entropy(h) == pytest.approx(ex["bits"], abs=1e-12)


def test_histogram_sum_and_permutation_invariance():
    s = eqsynth.random_codes_stream(100003, 1)
    h = o.histogram(s)
    assert int(h.sum()) == s.size
    assert (h == np.bincount(s, minlength=256).astype(np.uint64)).all()
    assert (o.histogram(np.random.default_rng(0).permutation(s)) == h).all()


# ------------------------------------------------------------------ table normalisation
def test_normalize_spec_examples(golden):
    ex = golden["spec_examples"]["normalize"]
    f = o.normalize(hist_of(ex[0]["counts"]))
    assert f[65] == 3072 and f[66] == 1024 and f.sum() == 4096
    f = o.normalize(hist_of(ex[1]["counts"]))
    assert f[7] == 4096 and f.sum() == 4096
    f = o.normalize(np.ones(256, dtype=np.uint64))
    assert (f == 16).all()


@pytest.mark.parametrize("k", [130, 248, 253, 255, 3, 1])
def test_normalize_uniform_subsets_never_invalid(k):
    """The SPEC literal rule goes negative on uniform-over-248/130."""
    h = np.zeros(256, dtype=np.uint64)
    h[np.random.default_rng(k).permutation(256)[:k]] = 1000
    f = o.normalize(h)
    assert f.sum() == 4096
    assert ((f >= 1) == (h > 0)).all()


def test_normalize_random_properties():
    rng = np.random.default_rng(7)
    for t in range(300):
        k = int(rng.integers(1, 257))
        h = np.zeros(256, dtype=np.uint64)
        idx = rng.permutation(256)[:k]
        h[idx] = (rng.pareto(1.0 + rng.uniform(0, 3), k) * 1000).astype(np.uint64) + 1
        f = o.normalize(h)
        assert f.sum() == 4096
        assert ((f >= 1) == (h > 0)).all()
        ideal = 4096 * h.astype(np.float64) / h.sum()
        if (ideal[h > 0] >= 1).all():
            # no symbol is lifted to 1, so D >= 0: every f is ⌊ideal⌋ or ⌊ideal⌋+1
            fl = np.floor(ideal)
            assert ((f == fl) | (f == fl + 1))[h > 0].all()
        # cross-entropy penalty of the table is small relative to Ĥ
        if h.sum() > 10000:
            assert xent_bits(h, f) <= emp_entropy_bits(h) + 0.06 * h.sum() + 1e-6


def _expand(d: dict) -> dict:
    """{"5": v, "100..399": v} -> {5: v, 100: v, ..., 399: v} (golden shorthand)."""
    out = {}
    for k, v in d.items():
        if ".." in k:
            a, b = (int(x) for x in k.split(".."))
            out.update({c: v for c in range(a, b + 1)})
        else:
            out[int(k)] = v
    return out


def test_normalize_worked_examples(golden):
    """Hand-derived R8 tables (tests/golden/normalize_worked.json): D > 0 with remainder, count
    and code tie-breaks; D < 0 with two give-back candidates that interleave, and an odd split."""
    for case in golden["normalize_worked"]["cases"]:
        f = o.normalize(hist_of(_expand(case["counts"])))
        want = np.zeros(256, np.int64)
        for c, v in _expand(case["freq"]).items():
            want[c] = v
        assert (f.astype(np.int64) == want).all(), case["name"]


def _r8_reference_parts(h):
    """floor / remainder of 4096·c/T in exact integers (Python ints, independent of the oracle)."""
    T = int(h.sum())
    q = {c: max(1, 4096 * int(h[c]) // T) for c in range(256) if h[c]}
    r = {c: (4096 * int(h[c])) % T for c in range(256) if h[c]}
    return q, r


def test_normalize_selection_properties():
    """Which symbols the R8 rule adjusts, checked against exact integer floors/remainders:
    D > 0 — exactly D present symbols get +1 and each of them ranks (r, c, -code) above every
    present symbol that did not; D < 0 — only symbols with f > 1 lose, and the losers end at
    the final maximum or one below it (take-from-the-largest water-filling)."""
    rng = np.random.default_rng(11)
    seen_pos = seen_neg = 0
    for t in range(400):
        k = int(rng.integers(2, 257))
        h = np.zeros(256, dtype=np.uint64)
        idx = rng.permutation(256)[:k]
        h[idx] = (rng.pareto(0.5 + rng.uniform(0, 3), k) * rng.choice([3, 30, 3000])).astype(np.uint64) + 1
        if t % 3 == 0:                      # many count-1 symbols under a heavy head: D < 0
            h[idx[: k // 2]] = 1
            h[idx[0]] += np.uint64(rng.integers(4096, 40000))
        f = o.normalize(h).astype(np.int64)
        q, r = _r8_reference_parts(h)
        D = 4096 - sum(q.values())
        pres = sorted(q)
        if D > 0:
            seen_pos += 1
            up = [c for c in pres if f[c] == q[c] + 1]
            assert len(up) == D and all(f[c] in (q[c], q[c] + 1) for c in pres)
            key = lambda c: (r[c], int(h[c]), -c)
            rest = [c for c in pres if f[c] == q[c]]
            if rest:
                assert min(key(c) for c in up) > max(key(c) for c in rest)
        elif D < 0:
            seen_neg += 1
            down = [c for c in pres if f[c] < q[c]]
            m = int(f.max())
            assert all(q[c] > 1 and f[c] >= max(m - 1, 1) for c in down)
            assert all(q[c] <= m for c in pres if c not in down)
            assert all(f[c] == q[c] for c in pres if c not in down)
        else:
            assert all(f[c] == q[c] for c in pres)
    assert seen_pos > 50 and seen_neg > 20


def test_pair_table_worked_examples(golden):
    """Hand-derived pair tables (R15): ranks with a count tie, D > 0 over pair weights (largest
    remainder), and a dropped pair with an escape and D < 0."""
    for case in golden["normalize_worked"]["pair_cases"]:
        pt = o.pair_table(hist_of(_expand(case["counts"])))
        assert pt.K == case["K"], case["name"]
        assert list(pt.rank_code[:pt.K]) == case["rank_code"], case["name"]
        want = np.zeros(225, np.int64)
        for k, v in case["pairs"].items():
            ra, rb = (int(x) for x in k.split(","))
            want[ra * 15 + rb] = v
        assert (pt.pf.astype(np.int64) == want).all(), case["name"]
        assert pt.fesc == case["fesc"], case["name"]


def test_pair_codec_worked_streams(golden):
    """Hand-derived pair-codec chunks (tests/golden/rans_pair_worked.json): an escaped pair, a kept
    pair and an odd tail; and a renormalisation-free two-pair chunk."""
    for case in golden["rans_pair_worked"]["cases"]:
        h = hist_of(_expand(case["counts"]))
        f = o.normalize(h)
        want = np.zeros(256, np.int64)
        for c, v in _expand(case["single_freq"]).items():
            want[c] = v
        assert (f.astype(np.int64) == want).all(), case["name"]
        pt = o.pair_table(h)
        sym = np.array(case["symbols"], dtype=np.uint8)
        data = o.encode_chunk_pair(sym, f, pt)
        assert data.hex() == case["bytes_hex"], case["name"]
        assert (o.decode_chunk_pair(data, f, pt, sym.size) == sym).all()


# ------------------------------------------------------------------ rANS chunks
CODECS = [o.CODEC_BYTE, o.CODEC_WORD]
GOLDEN_STREAMS = {o.CODEC_BYTE: "rans_worked", o.CODEC_WORD: "rans_word_worked"}
L_OF = {o.CODEC_BYTE: 1 << 23, o.CODEC_WORD: 1 << 16}


@pytest.mark.parametrize("codec", CODECS)
def test_rans_worked_examples(golden, codec):
    for case in golden[GOLDEN_STREAMS[codec]]["cases"]:
        freq = np.zeros(256, dtype=np.uint16)
        for k, v in case["freq"].items():
            freq[int(k)] = v
        sym = np.array(case["symbols"], dtype=np.uint8)
        data = o.encode_chunk(sym, freq, codec)
        assert data.hex() == case["bytes_hex"], case["name"]
        assert (o.decode_chunk(data, freq, sym.size, codec) == sym).all()


@pytest.mark.parametrize("codec", CODECS)
@pytest.mark.parametrize("kind", ["skewed", "uniform", "subset130", "subset248", "subset2", "single"])
def test_rans_round_trip_fuzz(kind, codec):
    rng = np.random.default_rng(hash(kind) & 0xFFFF)
    for t in range(25):
        n = int(rng.choice([0, 1, 2, 3, 17, 4095, 4096, 4097, int(rng.integers(1, 70000))]))
        s = eqsynth.random_codes_stream(max(n, 1), int(rng.integers(1 << 30)), kind)[:n]
        freq = o.normalize(o.histogram(s)) if n else o.normalize(np.ones(256, np.uint64))
        data = o.encode_chunk(s, freq, codec)
        assert (o.decode_chunk(data, freq, n, codec) == s).all()
        if codec == o.CODEC_WORD:
            assert len(data) % 2 == 0                  # 4-byte state + whole 16-bit words


@pytest.mark.parametrize("codec", CODECS)
def test_rans_empty_chunk_is_state_only(codec):
    freq = o.normalize(np.ones(256, np.uint64))
    data = o.encode_chunk(np.zeros(0, np.uint8), freq, codec)
    assert data == L_OF[codec].to_bytes(4, "little")


def test_rans_word_uniform_closed_form():
    """Word codec, all 256 symbols at f = 16 (closed form, derived by hand): x = 16q + r
    codes to 4096q + r + 16s.  From x = L = 2^16 the state alternates between
    [2^16, 2^16 + 2^12) and [2^24, 2^24 + 2^20): a symbol coded from the lower range lands in
    the upper one without output; the next one finds x ≥ 2^20·16 = 2^24, emits one word and
    returns to the lower range.  So n symbols cost exactly 4 + 2·⌊n/2⌋ bytes."""
    freq = np.full(256, 16, dtype=np.uint16)
    rng = np.random.default_rng(3)
    for n in [1, 2, 3, 4, 5, 20, 1001, 2000]:
        s = rng.integers(0, 256, n).astype(np.uint8)
        data = o.encode_chunk(s, freq, o.CODEC_WORD)
        assert len(data) == 4 + 2 * (n // 2)
        assert (o.decode_chunk(data, freq, s.size, o.CODEC_WORD) == s).all()


@pytest.mark.parametrize("codec", CODECS)
def test_rans_rate_bounds(codec):
    """Shannon lower bound and the table cross-entropy upper bound."""
    for kind, seed in [("skewed", 1), ("uniform", 2), ("subset40", 3)]:
        s = eqsynth.random_codes_stream(1 << 18, seed, kind)
        h = o.histogram(s)
        f = o.normalize(h)
        data = o.encode_chunk(s, f, codec)
        bits = 8 * len(data)
        assert bits >= emp_entropy_bits(h) - 0.001 * s.size
        assert bits <= xent_bits(h, f) + 0.01 * s.size + 64


@pytest.mark.parametrize("codec", CODECS)
def test_rans_degenerate_rates(codec):
    # 2^20 copies of one symbol -> < 0.01 bits/symbol
    s = np.full(1 << 20, 9, dtype=np.uint8)
    f = o.normalize(o.histogram(s))
    assert 8 * len(o.encode_chunk(s, f, codec)) / s.size < 0.01
    # uniform random bytes -> within 1% above 8 bits/symbol
    s = eqsynth.random_codes_stream(1 << 20, 5, "uniform")
    f = o.normalize(o.histogram(s))
    r = 8 * len(o.encode_chunk(s, f, codec)) / s.size
    assert 8.0 - 0.01 <= r <= 8.0 * 1.01


@pytest.mark.parametrize("codec", CODECS)
def test_rans_unknown_symbol_and_corruption(codec):
    f = o.normalize(hist_of({1: 5, 2: 5}))
    with pytest.raises(ValueError, match="unknown-symbol"):
        o.encode_chunk(np.array([1, 3], np.uint8), f, codec)
    s = eqsynth.random_codes_stream(5000, 9, "skewed")
    f = o.normalize(o.histogram(s))
    data = bytearray(o.encode_chunk(s, f, codec))
    with pytest.raises(ValueError, match="truncated"):
        o.decode_chunk(bytes(data[:-4]), f, s.size, codec)
    with pytest.raises(ValueError, match="corrupt|truncated"):
        o.decode_chunk(bytes(data) + b"\0\0", f, s.size, codec)     # unconsumed trailing bytes
    detected = 0
    for pos in range(4, len(data), max(1, len(data) // 40)):
        d2 = bytearray(data)
        d2[pos] ^= 0x5A
        try:
            out = o.decode_chunk(bytes(d2), f, s.size, codec)
            detected += int(not (out == s).all())      # wrong output at least
        except ValueError:
            detected += 1
    assert detected >= 0.9 * len(range(4, len(data), max(1, len(data) // 40)))


# ------------------------------------------------------------------ block stream
@pytest.mark.parametrize("codec", CODECS)
def test_block_round_trip_ragged_layers(codec):
    """Layer-restart chunking with ragged shapes and a tiny chunk size."""
    layers = [eqsynth.weights(r, c, seed=1, layer=0, matrix=m) for m, (r, c) in
              enumerate([(37, 53), (1, 1), (64, 64), (5, 4097)])]
    for cs in [4096, 100, 1]:
        blk = o.quantize_encode(layers, lam=None, cs=cs, codec=codec)
        stream = o.decode_block(blk)
        assert (stream == blk.codes).all()
        sym0, ns = o.chunk_table(blk.layer_shapes, cs)
        assert ns.sum() == stream.size and blk.n_chunks == ns.size
        # chunk independence: any chunk decodes alone to its slice
        for k in [0, blk.n_chunks // 2, blk.n_chunks - 1]:
            a, b = int(blk.chunk_off[k]), int(blk.chunk_off[k + 1])
            out = o.decode_chunk(blk.payload[a:b], blk.freq, int(ns[k]), codec)
            assert (out == stream[int(sym0[k]):int(sym0[k]) + int(ns[k])]).all()
        deq = o.decode_dequant(blk)
        for W, S, D in zip(layers, blk.scales, deq):
            assert (D == o.dequant(o.quantize(W, S), S)).all()


def test_block_lambda0_rate_near_paper_anchor():
    """λ=0 (AbsMax FP8 + ANS) lands near the paper's ≈6.5 bits/param;
    SPEC's loose band [5.5, 7.5]."""
    layers = eqsynth.block_weights("llama-3.2-1b", 0)[:2]
    layers = [W[:256] for W in layers]
    blk = o.quantize_encode(layers, lam=None)
    assert 5.5 <= blk.effective_bits() <= 7.5
    H = o.entropy(blk.hist)
    coded = len(blk.payload) + 4 * (blk.n_chunks + 1)
    assert coded <= 1.02 * blk.n_params * H / 8                       # north_star 1.02x
    assert len(blk.payload) * 8 >= blk.n_params * H - 0.001 * blk.n_params


@pytest.mark.parametrize("codec", CODECS)
def test_block_two_bits_unique_codes_and_budget(codec):
    """At ~2 bits: many more than 4 unique codes (Table 1) and coded size within
    1.02x of n·Ĥ (north_star)."""
    W = eqsynth.weights(64, 1024, seed=2)
    blk = o.quantize_encode([W], lam=180.0, codec=codec)
    H = o.entropy(blk.hist)
    assert 1.3 < H < 3.0
    assert int((blk.hist > 0).sum()) > 12
    coded = len(blk.payload) + 4 * (blk.n_chunks + 1)
    assert coded <= 1.02 * blk.n_params * H / 8


# ------------------------------------------------------------------ pair codec (R15; round-2 groundwork)
def test_pair_table_rules():
    """Integer table rules: ranks by count (ties: lower code), pairs kept iff 32·M·c_a·c_b ≥ T²,
    the R8 rule over [kept pairs, escape] sums to M, escape present iff some pair is not
    kept; a single-symbol histogram gives one pair of frequency M."""
    h = hist_of({7: 10})
    pt = o.pair_table(h)
    assert pt.K == 1 and pt.rank_code[0] == 7 and pt.pf[0] == 4096 and pt.fesc == 0
    h = hist_of({3: 50, 9: 50, 200: 1})
    pt = o.pair_table(h)
    assert list(pt.rank_code[:3]) == [3, 9, 200]                      # tie 3/9 -> lower code first
    T = 101
    for ra in range(pt.K):
        for rb in range(pt.K):
            w = int(h[pt.rank_code[ra]]) * int(h[pt.rank_code[rb]])
            assert (pt.pf[ra * 15 + rb] > 0) == (32 * 4096 * w >= T * T)
    assert int(pt.pf.sum()) + pt.fesc == 4096 and pt.fesc == 0          # every pair kept: no escape
    h = hist_of({3: 50000, 9: 50000, 200: 1})                            # (200, 200) below 1/32 slot
    pt = o.pair_table(h)
    assert pt.pf[2 * 15 + 2] == 0 and pt.pf[0] > 0 and pt.fesc >= 1
    assert int(pt.pf.sum()) + pt.fesc == 4096
    # 20 equiprobable codes: only the top 15 are ranked; everything else escapes
    h = np.zeros(256, np.uint64)
    h[np.arange(20) * 7] = 1000
    pt = o.pair_table(h)
    assert pt.K == 15 and int(pt.pf.sum()) + pt.fesc == 4096 and (pt.pf > 0).sum() == 225


@pytest.mark.parametrize("kind", ["skewed", "uniform", "subset2", "single", "subset40"])
def test_pair_codec_round_trip_and_rate(kind):
    rng = np.random.default_rng(hash(kind) & 0xFFFF)
    for t in range(6):
        n = int(rng.choice([1, 2, 3, 17, 4095, 4097, int(rng.integers(1, 12000))]))
        s = eqsynth.random_codes_stream(n, int(rng.integers(1 << 30)), kind)
        h = o.histogram(s)
        f = o.normalize(h)
        pt = o.pair_table(h)
        data = o.encode_chunk_pair(s, f, pt)
        assert (o.decode_chunk_pair(data, f, pt, n) == s).all()
        assert 8 * len(data) >= emp_entropy_bits(h) - 0.001 * n - 32     # Shannon (i.i.d. pairs)
    with pytest.raises(ValueError):
        o.decode_chunk_pair(data[:-2], f, pt, n)


def test_pair_codec_block_rate_at_two_bits():
    """Pair coding of the bench's synthetic 2-bit weights: lossless, and within 1.5 % of the
    word codec's payload (the pair table's quantisation and the escapes cost ~1 %)."""
    W = eqsynth.weights(32, 4096, seed=2)
    S = o.search(W, 230.0)[0]
    bw = o.quantize_encode([W], scales=[S], codec=o.CODEC_WORD)
    bp = o.quantize_encode([W], scales=[S], codec=o.CODEC_PAIR)
    assert (o.decode_block(bp) == bp.codes).all()
    assert len(bp.payload) <= 1.015 * len(bw.payload)
    H = o.entropy(bp.hist)
    assert len(bp.payload) + 4 * (bp.n_chunks + 1) <= 1.02 * W.numel() * H / 8


def test_cpu_baseline_helpers_match_block_decode():
    """bench.py's multi-threaded CPU baseline decodes exactly what decode_dequant does (all
    three codecs): timing helper, same arithmetic."""
    W = eqsynth.weights(64, 1024, seed=9)
    S = (o.absmax_scales(W).astype(np.int32) + 1600).astype(np.uint16)
    for codec in (o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G):
        blk = o.quantize_encode([W], scales=[S], cs=512, codec=codec)
        payload = np.frombuffer(blk.payload + b"\0" * 16, dtype=np.uint8)
        out = o.decode_dequant_layer_mt(payload, blk.chunk_off, 512, 64, 1024, S, blk.freq, 3, codec, blk.pair)
        assert (out == o.decode_dequant(blk)[0]).all(), codec


# ------------------------------------------------------------------ grouped escapes (R18)
def test_pair_grouped_worked_streams(golden):
    """Hand-derived R18 chunk (tests/golden/rans_pair_worked.json): an escape BEFORE a kept pair
    of its group, so its two codes come after that pair — bytes differ from the R15 stream."""
    for case in golden["rans_pair_worked"]["grouped_cases"]:
        h = hist_of(_expand(case["counts"]))
        f = o.normalize(h)
        pt = o.pair_table(h)
        sym = np.array(case["symbols"], dtype=np.uint8)
        data = o.encode_chunk_pair(sym, f, pt, grouped=True)
        assert data.hex() == case["bytes_hex"], case["name"]
        assert (o.decode_chunk_pair(data, f, pt, sym.size, grouped=True) == sym).all()
        assert (o.encode_chunk_pair(sym, f, pt).hex() != data.hex()) == case["r15_bytes_hex_differs"]


def _escaped(sym, pt):
    rank = np.full(256, -1)
    rank[pt.rank_code[:pt.K]] = np.arange(pt.K)
    a, b = rank[sym[0:sym.size // 2 * 2:2]], rank[sym[1:sym.size // 2 * 2:2]]
    ok = (a >= 0) & (b >= 0)
    ok[ok] = pt.pf[a[ok] * 15 + b[ok]] > 0
    return ~ok


@pytest.mark.parametrize("n", [16, 17, 32, 33, 46, 64])
def test_pair_grouped_equals_r15_when_escapes_end_their_group(n):
    """When every escaped pair is the LAST pair position of its 16-symbol group, R18's decode
    order (group pairs, then the escaped codes, then an odd last symbol) is R15's order, so the
    two streams are byte-identical — a 32-symbol group, or escapes deferred to the chunk's end,
    would break this for n > 16."""
    rng = np.random.default_rng(n)
    h = np.zeros(256, np.uint64)
    h[0], h[1], h[2], h[3] = 1000, 10, 1, 1            # (2,2), (2,3), (3,2), (3,3) are escapes
    f, pt = o.normalize(h), o.pair_table(h)
    for t in range(20):
        sym = rng.choice(np.array([0, 0, 0, 1], np.uint8), n)
        for g0 in range(0, n, 16):
            last = min(g0 + 16, n) // 2 * 2 - 2       # the group's last pair position (symbol index)
            if last >= g0 and rng.random() < 0.7:
                sym[last], sym[last + 1] = rng.choice([2, 3]), rng.choice([2, 3])
        esc = _escaped(sym, pt)
        assert esc.any() or t > 0 or n < 16
        data = o.encode_chunk_pair(sym, f, pt, grouped=True)
        assert data == o.encode_chunk_pair(sym, f, pt)
        assert (o.decode_chunk_pair(data, f, pt, n, grouped=True) == sym).all()


@pytest.mark.parametrize("kind", ["skewed", "uniform", "subset2", "single", "subset40"])
def test_pair_grouped_round_trip_and_same_rate(kind):
    """R18 codes the same symbols as R15 with the same (f, c), only reordered: lossless, and
    the payloads differ by at most one 16-bit word (the final state's end effect); escapes
    anywhere, every length class (empty groups, odd tails, several groups)."""
    rng = np.random.default_rng((hash(kind) + 7) & 0xFFFF)
    for t in range(8):
        n = int(rng.choice([1, 2, 3, 15, 16, 17, 31, 4095, 4096, 4097, int(rng.integers(1, 12000))]))
        s = eqsynth.random_codes_stream(n, int(rng.integers(1 << 30)), kind)
        h = o.histogram(s)
        f = o.normalize(h)
        pt = o.pair_table(h)
        g = o.encode_chunk_pair(s, f, pt, grouped=True)
        r = o.encode_chunk_pair(s, f, pt)
        assert (o.decode_chunk_pair(g, f, pt, n, grouped=True) == s).all()
        assert abs(len(g) - len(r)) <= 2, (n, len(g), len(r))
    with pytest.raises(ValueError):
        o.decode_chunk_pair(g[:-2], f, pt, n, grouped=True)


def _word_rans_encode(steps):
    """R14's word rANS written out (pinned by tests/golden/rans_word_worked.json): encode the
    decode-order list of (f, c) steps backwards from x = L = 2^16; emit the low 16 bits while
    x ≥ 2^20·f; the 4-byte LE final state, then the words in decode order."""
    x, words = 1 << 16, []
    for f, c in reversed(steps):
        while x >= (1 << 20) * f:
            words.append(x & 0xFFFF)
            x >>= 16
        x = (x // f) * 4096 + x % f + c
    out = bytes([x & 0xFF, (x >> 8) & 0xFF, (x >> 16) & 0xFF, (x >> 24) & 0xFF])
    for w in reversed(words):
        out += bytes([w & 0xFF, w >> 8])
    return out


def _r18_steps(sym, f, pt):
    """R18 read literally: for each 16-symbol group of the chunk, in order — its
    pair positions (kept pair: the pair table's (f, c); else the escape's), then for each escaped
    position in increasing order the single-table (f, c) of its first then second code, then the
    group's odd last symbol."""
    cum = np.concatenate([[0], np.cumsum(f.astype(np.int64))])
    rank = {int(pt.rank_code[r]): r for r in range(pt.K)}
    pcum, run = {}, 0
    for q in range(225):
        if q // 15 < pt.K and q % 15 < pt.K and pt.pf[q]:
            pcum[q] = run
            run += int(pt.pf[q])
    cesc = run
    steps = []
    for g0 in range(0, sym.size, 16):
        grp = [int(v) for v in sym[g0:g0 + 16]]
        esc = []
        for i in range(len(grp) // 2):
            a, b = grp[2 * i], grp[2 * i + 1]
            q = rank[a] * 15 + rank[b] if a in rank and b in rank else None
            if q is not None and q in pcum:
                steps.append((int(pt.pf[q]), pcum[q]))
            else:
                steps.append((pt.fesc, cesc))
                esc.append(i)
        for i in esc:
            for s in (grp[2 * i], grp[2 * i + 1]):
                steps.append((int(f[s]), int(cum[s])))
        if len(grp) % 2:
            steps.append((int(f[grp[-1]]), int(cum[grp[-1]])))
    return steps


@pytest.mark.parametrize("kind", ["uniform", "subset40", "skewed"])
def test_pair_grouped_matches_the_literal_order(kind):
    """The C oracle's R18 stream equals R14's word coder run over the R18 decode order written out
    from its definition (several escapes per group, every length class): a wrong group size,
    escapes in decreasing order, or the odd symbol before the escaped codes would differ."""
    rng = np.random.default_rng((hash(kind) + 11) & 0xFFFF)
    for t in range(6):
        n = int(rng.choice([1, 3, 16, 17, 33, 47, 200, 4096, int(rng.integers(1, 3000))]))
        s = eqsynth.random_codes_stream(n, int(rng.integers(1 << 30)), kind)
        h = o.histogram(s)
        f = o.normalize(h)
        pt = o.pair_table(h)
        assert o.encode_chunk_pair(s, f, pt, grouped=True) == _word_rans_encode(_r18_steps(s, f, pt)), (kind, n)


def test_pair_grouped_decoder_rejects_the_r15_order():
    """The hand-derived R15 stream (escape at position 0, kept pair after it) read as R18 is not
    the same chunk: the integrity check (final state L, every word consumed) or the symbols
    differ — the two orders are distinguishable."""
    h = np.zeros(256, np.uint64)
    h[0], h[1], h[2], h[3] = 1000, 10, 1, 1
    f, pt = o.normalize(h), o.pair_table(h)
    sym = np.array([2, 3, 0, 1, 0], np.uint8)
    r15 = o.encode_chunk_pair(sym, f, pt)
    try:
        got = o.decode_chunk_pair(r15, f, pt, 5, grouped=True)
        assert not (got == sym).all()
    except ValueError:
        pass


# ------------------------------------------------------------------ EQ_CHUNK_ROW
ALL_CODECS = [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G]


def _chunk_alone(blk, k, n):
    data = blk.payload[int(blk.chunk_off[k]):int(blk.chunk_off[k + 1])]
    if blk.codec in o.PAIR_CODECS:
        return o.decode_chunk_pair(data, blk.freq, blk.pair, n, grouped=blk.codec == o.CODEC_PAIR_G)
    return o.decode_chunk(data, blk.freq, n, blk.codec)


@pytest.mark.parametrize("codec", ALL_CODECS)
def test_row_chunking_layout_by_brute_force(codec):
    """Row chunking: a row of K columns is ⌈K/cs⌉ chunks (full chunks, then the remainder);
    chunk k, decoded ALONE from its byte range, is exactly the codes of its (row, column
    range) — 10 columns at cs = 4 give 4 + 4 + 2, 7 columns give 4 + 3."""
    rng = np.random.default_rng(codec)
    shapes = [(6, 10), (3, 7), (2, 4)]
    codes = [eqsynth.random_codes_stream(r * c, int(rng.integers(1 << 30)), "skewed").reshape(r, c) for r, c in shapes]
    S = [np.full(r, 0x3F80, np.uint16) for r, _ in shapes]
    blk = o.encode_codes(codes, shapes, S, 4, codec=codec, chunk_mode=o.CHUNK_ROW)
    assert blk.n_chunks == 6 * 3 + 3 * 2 + 2 * 1
    k = 0
    for C, (r, c) in zip(codes, shapes):
        for row in range(r):
            for j0 in range(0, c, 4):
                want = C[row, j0:min(c, j0 + 4)]
                assert (_chunk_alone(blk, k, want.size) == want).all(), (k, row, j0)
                k += 1
    assert k == blk.n_chunks
    assert (o.decode_block(blk) == np.concatenate([C.reshape(-1) for C in codes])).all()
    assert (blk.codes == np.concatenate([C.reshape(-1) for C in codes])).all()      # layer order


@pytest.mark.parametrize("codec", ALL_CODECS)
def test_row_chunking_equals_layer_chunking_when_rows_are_whole_chunks(codec):
    """K % cs == 0: row boundaries already are chunk boundaries, so the two modes give the
    same bytes (the Llama-3-8B layers with K = 4096 at cs = 4096 / 2048)."""
    W = eqsynth.weights(24, 512, seed=3)
    S = (o.absmax_scales(W).astype(np.int32) + 1700).astype(np.uint16)
    a = o.quantize_encode([W], scales=[S], cs=256, codec=codec)
    b = o.quantize_encode([W], scales=[S], cs=256, codec=codec, chunk_mode=o.CHUNK_ROW)
    assert a.payload == b.payload and (a.chunk_off == b.chunk_off).all()


@pytest.mark.parametrize("codec", ALL_CODECS)
def test_row_chunking_threaded_dequant_helper(codec):
    """The threaded decode + dequant helper (bench CPU baseline, full-size parity) follows the
    row layout: equal to decode_dequant for K = 700 at cs = 256 (256 + 256 + 188 per row)."""
    W = eqsynth.weights(40, 700, seed=5)
    S = (o.absmax_scales(W).astype(np.int32) + 1600).astype(np.uint16)
    blk = o.quantize_encode([W], scales=[S], cs=256, codec=codec, chunk_mode=o.CHUNK_ROW)
    assert blk.n_chunks == 40 * 3
    payload = np.frombuffer(blk.payload + b"\0" * 16, dtype=np.uint8)
    out = o.decode_dequant_layer_mt(payload, blk.chunk_off, 256, 40, 700, S, blk.freq, 3, codec, blk.pair,
                                    chunk_mode=o.CHUNK_ROW)
    assert (out == o.decode_dequant(blk)[0]).all()


# ------------------------------------------------------------------ CHUNK_INTERLEAVED (R17)
def _interleave_literal(size: int, cs: int) -> list:
    """R17 read literally: for each whole super-chunk of 32·cs symbols, chunk j holds the
    super-chunk's 16-symbol groups j, j + 32, j + 64, …; the rest of the layer is plain
    chunks.  Returns, per chunk, the list of layer positions of its symbols in order."""
    chunks, sc = [], 32 * cs
    full = size // sc
    for s in range(full):
        for j in range(32):
            pos = []
            for g in range(j, cs // 16 * 32, 32):            # groups j, j + 32, … of the super-chunk
                pos.extend(range(s * sc + g * 16, s * sc + g * 16 + 16))
            chunks.append(pos)
    for a in range(full * sc, size, cs):
        chunks.append(list(range(a, min(size, a + cs))))
    return chunks


@pytest.mark.parametrize("size,cs", [(3 * 32 * 32 + 100, 32), (32 * 64, 64), (1000, 48), (2 * 32 * 48 + 48, 48)])
def test_interleave_order_matches_the_literal_definition(size, cs):
    lit = _interleave_literal(size, cs)
    src = o.interleave_order(size, cs)
    assert np.array_equal(np.sort(src), np.arange(size))                 # a permutation
    assert np.array_equal(src, np.concatenate([np.array(c, dtype=np.int64) for c in lit]))
    assert len(lit) == (size + cs - 1) // cs                            # as many chunks as layer chunking


@pytest.mark.parametrize("codec", ALL_CODECS)
def test_interleaved_chunking_layout_by_brute_force(codec):
    """Each chunk, decoded ALONE from its byte range, is exactly the codes at its R17 positions
    (whole super-chunks interleaved, then a ragged tail of plain chunks); the block round trips."""
    rng = np.random.default_rng(10 + codec)
    shapes = [(8, 272), (3, 80), (5, 16)]                               # cs 32: 2176 = 2·1024 + 128, 240, 80
    codes = [eqsynth.random_codes_stream(r * c, int(rng.integers(1 << 30)), "skewed").reshape(r, c) for r, c in shapes]
    S = [np.full(r, 0x3F80, np.uint16) for r, _ in shapes]
    blk = o.encode_codes(codes, shapes, S, 32, codec=codec, chunk_mode=o.CHUNK_INTERLEAVED)
    k = 0
    for C, (r, c) in zip(codes, shapes):
        flat = C.reshape(-1)
        for pos in _interleave_literal(r * c, 32):
            want = flat[np.array(pos)]
            assert (_chunk_alone(blk, k, want.size) == want).all(), (k, pos[:3])
            k += 1
    assert k == blk.n_chunks
    assert (o.decode_block(blk) == np.concatenate([C.reshape(-1) for C in codes])).all()
    assert (blk.codes == np.concatenate([C.reshape(-1) for C in codes])).all()      # layer order


@pytest.mark.parametrize("codec", ALL_CODECS)
def test_interleaved_chunking_degenerate_cases(codec):
    """A layer shorter than one super-chunk is plain layer chunking; with cs = 16 every chunk is
    one group, so R17 is layer chunking too — the same bytes in both cases.  A layer of whole
    super-chunks has the same chunk count and, for i.i.d. symbols, the same rate up to rANS state
    effects (the symbols of each chunk differ, the table does not)."""
    W = eqsynth.weights(24, 512, seed=13)
    S = (o.absmax_scales(W).astype(np.int32) + 1700).astype(np.uint16)
    for cs in (1024, 16):                                                # 24·512 < 32·1024; cs 16: groups = chunks
        a = o.quantize_encode([W], scales=[S], cs=cs, codec=codec)
        b = o.quantize_encode([W], scales=[S], cs=cs, codec=codec, chunk_mode=o.CHUNK_INTERLEAVED)
        assert a.payload == b.payload and (a.chunk_off == b.chunk_off).all(), cs
    a = o.quantize_encode([W], scales=[S], cs=128, codec=codec)
    b = o.quantize_encode([W], scales=[S], cs=128, codec=codec, chunk_mode=o.CHUNK_INTERLEAVED)
    assert a.n_chunks == b.n_chunks and a.payload != b.payload
    assert abs(len(a.payload) - len(b.payload)) <= 0.01 * len(a.payload)
    assert (o.decode_block(b) == o.decode_block(a)).all()


@pytest.mark.parametrize("codec", ALL_CODECS)
def test_interleaved_chunking_threaded_dequant_helper(codec):
    """The threaded decode + dequant helper follows R17: equal to decode_dequant (per-row scales
    spread over the interleaved groups)."""
    W = eqsynth.weights(40, 704, seed=15)
    S = (o.absmax_scales(W).astype(np.int32) + 1600).astype(np.uint16)
    blk = o.quantize_encode([W], scales=[S], cs=256, codec=codec, chunk_mode=o.CHUNK_INTERLEAVED)
    payload = np.frombuffer(blk.payload + b"\0" * 16, dtype=np.uint8)
    out = o.decode_dequant_layer_mt(payload, blk.chunk_off, 256, 40, 704, S, blk.freq, 3, codec, blk.pair,
                                    chunk_mode=o.CHUNK_INTERLEAVED)
    assert (out == o.decode_dequant(blk)[0]).all()


# ------------------------------------------------------------------ CRC verify mode
def test_crc32_check_values():
    """CRC-32/IEEE's catalogued check value ("123456789" → 0xCBF43926) and the empty message;
    a bit-by-bit long division with the reflected polynomial on short random strings."""
    assert o.crc32(np.frombuffer(b"123456789", np.uint8)) == 0xCBF43926
    assert o.crc32(np.zeros(0, np.uint8)) == 0

    def bitwise(b):
        c = 0xFFFFFFFF
        for byte in b:
            c ^= int(byte)
            for _ in range(8):
                c = (c >> 1) ^ (0xEDB88320 if c & 1 else 0)
        return c ^ 0xFFFFFFFF
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 64, 333):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        assert o.crc32(b) == bitwise(b)
