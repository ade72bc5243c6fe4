"""CPU oracle for the EntQuant hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2601_22787_b200`` never imports it and shares no code with it.

The arithmetic lives in ``eq_oracle.c`` (plain C, fp64, one function per paper step,
each citing PAPER.md / SPEC.md lines).  This module only marshals numpy arrays into it
and composes the steps in Alg. 1 / Alg. 2 order.

Parity status per function: every function here is pinned by a
``-m "not gpu"`` test in tests/test_oracle_*.py except ``search`` at λ's absolute scale,
which is "parity unpinned" for the paper's L-BFGS trajectory (only the exhaustive
reading is pinned, by brute force on tiny tensors and by the special cases).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eq_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

PROB_BITS = 12
CHUNK_SYMBOLS = 4096
FMT_E4M3, FMT_INT8 = 0, 1
CODEC_BYTE, CODEC_WORD = 0, 1      # rANS renormalisation: bytes (R9) / 16-bit words (R14)
CODEC_PAIR = 2                      # word rANS over pairs of symbols with escapes (R15)
CODEC_PAIR_G = 3                    # the same with each 16-symbol group's escaped codes after its pairs (R18)
PAIR_CODECS = (CODEC_PAIR, CODEC_PAIR_G)
CHUNK_LAYER, CHUNK_ROW = 0, 1       # chunks restart at every layer start / also at every row start (§8c.10)
CHUNK_INTERLEAVED = 2                # R17: layer chunking over 16-symbol groups dealt to 32 chunks in turn
IL_GROUP, IL_WAYS = 16, 32
PAIR_K = 15


def build(force: bool = False) -> str:
    """Compile eq_oracle.c with gcc (plain -O2, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", "-o", _SO, _SRC, "-lm", "-lpthread"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64, i32, u16, u32, dbl = (ctypes.c_int64, ctypes.c_int32, ctypes.c_uint16,
                                   ctypes.c_uint32, ctypes.c_double)
        sig = {
            "eqo_e4m3_value": (dbl, [u32]),
            "eqo_bf16_to_double": (dbl, [u16]),
            "eqo_bf16_from_double": (u16, [dbl]),
            "eqo_quantize_value": (ctypes.c_uint8, [dbl]),
            "eqo_quantize_value_scan": (ctypes.c_uint8, [dbl]),
            "eqo_quantize_one": (ctypes.c_uint8, [u16, u16]),
            "eqo_absmax_scale": (u16, [P, i64]),
            "eqo_quantize": (None, [P, i64, i64, P, P]),
            "eqo_dequant": (None, [P, i64, i64, P, P]),
            "eqo_row_terms": (None, [P, i64, u16, P, P]),
            "eqo_l1": (dbl, [P, i64]),
            "eqo_objective": (dbl, [P, i64, i64, P, dbl]),
            "eqo_candidates": (i64, [u16, i32, i32, P]),
            "eqo_search_rows": (None, [P, i64, i64, dbl, i32, i32, i64, i64, P, P]),
            "eqo_row_objectives": (i64, [P, i64, i64, i64, dbl, i32, i32, P, P, i64]),
            "eqo_qmax": (dbl, [ctypes.c_int]),
            "eqo_grid_value": (dbl, [ctypes.c_int, u32]),
            "eqo_grid_quantize": (ctypes.c_uint8, [ctypes.c_int, dbl]),
            "eqo_absmax_scale_fmt": (u16, [ctypes.c_int, P, i64]),
            "eqo_quantize_fmt": (None, [ctypes.c_int, P, i64, i64, P, P]),
            "eqo_dequant_fmt": (None, [ctypes.c_int, P, i64, i64, P, P]),
            "eqo_row_terms_fmt": (None, [ctypes.c_int, P, i64, u16, P, P]),
            "eqo_rd_row_fmt": (None, [ctypes.c_int, P, i64, u16, P]),
            "eqo_objective_fmt": (dbl, [ctypes.c_int, P, i64, i64, P, dbl]),
            "eqo_search_rows_fmt": (None, [ctypes.c_int, P, i64, i64, dbl, i32, i32, i64, i64, P, P]),
            "eqo_row_objectives_fmt": (i64, [ctypes.c_int, P, i64, i64, i64, dbl, i32, i32, P, P, i64]),
            "eqo_histogram": (None, [P, i64, P]),
            "eqo_normalize": (ctypes.c_int, [P, P]),
            "eqo_entropy": (dbl, [P]),
            "eqo_encode_chunk": (i64, [P, i64, P, P, i64]),
            "eqo_decode_chunk": (ctypes.c_int, [P, i64, P, P, i64]),
            "eqo_block_chunks": (i64, [P, i32, i64]),
            "eqo_encode_block": (i64, [P, P, i32, i64, P, P, i64, P]),
            "eqo_decode_block": (ctypes.c_int, [P, P, P, i32, i64, P, P]),
            "eqo_decode_chunks_mt": (ctypes.c_int, [P, P, P, P, i64, P, P, ctypes.c_int]),
            "eqo_decode_dequant_layer_mt": (ctypes.c_int, [P, P, i64, i64, i64, i64, P, P, P, ctypes.c_int]),
            "eqo_encode_chunk_codec": (i64, [ctypes.c_int, P, i64, P, P, i64]),
            "eqo_decode_dequant_layer_mt_pair": (ctypes.c_int, [P, P, i64, i64, i64, i64, P, P, P, i32, P, u16, P,
                                                                ctypes.c_int]),
            "eqo_pair_table": (ctypes.c_int, [P, P, P, P, P]),
            "eqo_encode_chunk_pair": (i64, [P, i64, P, P, i32, P, u16, P, i64]),
            "eqo_decode_chunk_pair": (ctypes.c_int, [P, i64, P, P, i32, P, u16, P, i64]),
            "eqo_encode_block_pair": (i64, [P, P, i32, i64, P, P, i32, P, u16, P, i64, P]),
            "eqo_decode_block_pair": (ctypes.c_int, [P, P, P, i32, i64, P, P, i32, P, u16, P]),
            "eqo_decode_chunk_codec": (ctypes.c_int, [ctypes.c_int, P, i64, P, P, i64]),
            "eqo_encode_block_codec": (i64, [ctypes.c_int, P, P, i32, i64, P, P, i64, P]),
            "eqo_decode_block_codec": (ctypes.c_int, [ctypes.c_int, P, P, P, i32, i64, P, P]),
            "eqo_decode_chunks_mt_codec": (ctypes.c_int, [ctypes.c_int, P, P, P, P, i64, P, P, ctypes.c_int]),
            "eqo_decode_dequant_layer_mt_codec": (ctypes.c_int, [ctypes.c_int, P, P, i64, i64, i64, i64, P, P, P,
                                                                 ctypes.c_int]),
            "eqo_decode_dequant_layer_mt_codec_seg": (ctypes.c_int, [ctypes.c_int, P, P, i64, i64, i64, i64, i64, P, P,
                                                                     P, ctypes.c_int]),
            "eqo_decode_dequant_layer_mt_pair_seg": (ctypes.c_int, [P, P, i64, i64, i64, i64, i64, P, P, P, i32, P, u16,
                                                                    P, ctypes.c_int]),
            "eqo_encode_chunk_pairg": (i64, [P, i64, P, P, i32, P, u16, P, i64]),
            "eqo_decode_chunk_pairg": (ctypes.c_int, [P, i64, P, P, i32, P, u16, P, i64]),
            "eqo_encode_block_pairx": (i64, [P, P, i32, i64, P, P, i32, P, u16, P, i64, P, i32]),
            "eqo_decode_block_pairx": (ctypes.c_int, [P, P, P, i32, i64, P, P, i32, P, u16, P, i32]),
            "eqo_decode_dequant_layer_mt_pairx_seg": (ctypes.c_int, [P, P, i64, i64, i64, i64, i64, P, P, P, i32, P,
                                                                     u16, P, ctypes.c_int, i32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def _u16(a) -> np.ndarray:
    """bf16 bit patterns as uint16 (accepts torch bf16 tensors or uint16 arrays)."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return np.ascontiguousarray(a.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16))
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint16))


# ---------------------------------------------------------------- scalar steps
def e4m3_value(code: int) -> float:
    return lib().eqo_e4m3_value(code)


def bf16_to_float(b: int) -> float:
    return lib().eqo_bf16_to_double(b)


def bf16_from_float(x: float) -> int:
    return lib().eqo_bf16_from_double(x)


def quantize_value(r: float) -> int:
    return lib().eqo_quantize_value(r)


def quantize_value_scan(r: float) -> int:
    return lib().eqo_quantize_value_scan(r)


def quantize_one(w_bf16: int, s_bf16: int) -> int:
    return lib().eqo_quantize_one(w_bf16, s_bf16)


# ---------------------------------------------------------------- matrix steps
def grid_value(code: int, fmt: int = FMT_E4M3) -> float:
    return lib().eqo_grid_value(fmt, code)


def grid_quantize(r: float, fmt: int = FMT_E4M3) -> int:
    return lib().eqo_grid_quantize(fmt, r)


def absmax_scales(W, fmt: int = FMT_E4M3) -> np.ndarray:
    """Eq. (1), Alg. 1 l.1: per-row AbsMax scale as bf16 bits."""
    W = _u16(W)
    M, N = W.shape
    return np.array([lib().eqo_absmax_scale_fmt(fmt, _p(W[i]), N) for i in range(M)], dtype=np.uint16)


def quantize(W, S, fmt: int = FMT_E4M3) -> np.ndarray:
    """Alg. 1 l.3: codes = Q_γ(W, S)."""
    W, S = _u16(W), _u16(S)
    M, N = W.shape
    out = np.empty((M, N), dtype=np.uint8)
    lib().eqo_quantize_fmt(fmt, _p(W), M, N, _p(S), _p(out))
    return out


def dequant(codes: np.ndarray, S, fmt: int = FMT_E4M3) -> np.ndarray:
    """Q†: bf16 bits of RNE(s·value(code))."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    S = _u16(S)
    M, N = codes.shape
    out = np.empty((M, N), dtype=np.uint16)
    lib().eqo_dequant_fmt(fmt, _p(codes), M, N, _p(S), _p(out))
    return out


def row_terms(w_row, s_bf16: int, fmt: int = FMT_E4M3):
    w_row = _u16(w_row)
    D, R = ctypes.c_double(), ctypes.c_double()
    lib().eqo_row_terms_fmt(fmt, _p(w_row), w_row.size, s_bf16, ctypes.byref(D), ctypes.byref(R))
    return D.value, R.value


def rd_row(w_row, s_bf16: int, fmt: int = FMT_E4M3) -> np.ndarray:
    """Row sums {D, R, A, B, Q} of Eq. 4 and its straight-through derivative (eqo_rd_row_fmt)."""
    w_row = _u16(w_row)
    out = np.zeros(5, dtype=np.float64)
    lib().eqo_rd_row_fmt(fmt, _p(w_row), w_row.size, int(s_bf16), _p(out))
    return out


def l1(W) -> float:
    W = _u16(W)
    return lib().eqo_l1(_p(W), W.size)


def objective(W, S, lam: float, fmt: int = FMT_E4M3) -> float:
    W, S = _u16(W), _u16(S)
    M, N = W.shape
    return lib().eqo_objective_fmt(fmt, _p(W), M, N, _p(S), lam)


def candidates(s0: int, oct_lo: int = -1, oct_hi: int = 20):
    first = ctypes.c_uint16()
    n = lib().eqo_candidates(s0, oct_lo, oct_hi, ctypes.byref(first))
    return first.value, n


def search(W, lam: float, oct_lo: int = -1, oct_hi: int = 20, rows=None, fmt: int = FMT_E4M3):
    """Alg. 1 l.2 (exhaustive per-row reading): returns (S bf16 bits, per-row objective).

    ``rows`` optionally restricts the search to a list of row indices (others are 0)."""
    W = _u16(W)
    M, N = W.shape
    S = np.zeros(M, dtype=np.uint16)
    f = np.zeros(M, dtype=np.float64)
    if rows is None:
        lib().eqo_search_rows_fmt(fmt, _p(W), M, N, lam, oct_lo, oct_hi, 0, M, _p(S), _p(f))
    else:
        for r in rows:
            lib().eqo_search_rows_fmt(fmt, _p(W), M, N, lam, oct_lo, oct_hi, int(r), int(r) + 1, _p(S), _p(f))
    return S, f


def row_objectives(W, row: int, lam: float, oct_lo: int = -1, oct_hi: int = 20, fmt: int = FMT_E4M3):
    """All candidate objectives f_i(s) of one row: (first pattern, array)."""
    W = _u16(W)
    M, N = W.shape
    cap = 128 * (oct_hi - oct_lo) + 8
    f = np.zeros(cap, dtype=np.float64)
    first = ctypes.c_uint16()
    n = lib().eqo_row_objectives_fmt(fmt, _p(W), M, N, row, lam, oct_lo, oct_hi, ctypes.byref(first), _p(f), cap)
    return first.value, f[:n].copy()


def histogram(sym: np.ndarray) -> np.ndarray:
    sym = np.ascontiguousarray(sym, dtype=np.uint8).reshape(-1)
    h = np.zeros(256, dtype=np.uint64)
    lib().eqo_histogram(_p(sym), sym.size, _p(h))
    return h


def normalize(hist: np.ndarray) -> np.ndarray:
    hist = np.ascontiguousarray(hist, dtype=np.uint64)
    f = np.zeros(256, dtype=np.uint16)
    if lib().eqo_normalize(_p(hist), _p(f)) != 0:
        raise ValueError("empty")
    return f


def entropy(hist: np.ndarray) -> float:
    hist = np.ascontiguousarray(hist, dtype=np.uint64)
    return lib().eqo_entropy(_p(hist))


def encode_chunk(sym: np.ndarray, freq: np.ndarray, codec: int = CODEC_BYTE) -> bytes:
    sym = np.ascontiguousarray(sym, dtype=np.uint8).reshape(-1)
    freq = np.ascontiguousarray(freq, dtype=np.uint16)
    cap = 4 + 2 * sym.size + 8
    out = np.zeros(cap, dtype=np.uint8)
    n = lib().eqo_encode_chunk_codec(codec, _p(sym), sym.size, _p(freq), _p(out), cap)
    if n == -2:
        raise ValueError("unknown-symbol")
    if n < 0:
        raise ValueError("buffer")
    return out[:n].tobytes()


def decode_chunk(data: bytes, freq: np.ndarray, n: int, codec: int = CODEC_BYTE) -> np.ndarray:
    buf = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    freq = np.ascontiguousarray(freq, dtype=np.uint16)
    out = np.zeros(max(n, 1), dtype=np.uint8)
    st = lib().eqo_decode_chunk_codec(codec, _p(buf), len(data), _p(freq), _p(out), n)
    if st == 1:
        raise ValueError("corrupt")
    if st == 2:
        raise ValueError("truncated")
    return out[:n]


@dataclass
class PairTable:
    """Tables of the pair codec (R15): rank_code uint8[16], K ranked codes, pf uint16[225]
    pair frequencies by (ra, rb) = ra*15 + rb (0 = not kept), fesc escape frequency."""
    rank_code: np.ndarray
    K: int
    pf: np.ndarray
    fesc: int


def pair_table(hist: np.ndarray) -> PairTable:
    hist = np.ascontiguousarray(hist, dtype=np.uint64)
    rc = np.zeros(16, dtype=np.uint8)
    K = ctypes.c_int32()
    pf = np.zeros(225, dtype=np.uint16)
    fe = ctypes.c_uint16()
    if lib().eqo_pair_table(_p(hist), _p(rc), ctypes.byref(K), _p(pf), ctypes.byref(fe)) != 0:
        raise ValueError("empty")
    return PairTable(rc, K.value, pf, fe.value)


def encode_chunk_pair(sym: np.ndarray, freq: np.ndarray, pt: PairTable, grouped: bool = False) -> bytes:
    """One chunk of the pair codec: R15 order, or R18 (grouped escapes) when ``grouped``."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8).reshape(-1)
    freq = np.ascontiguousarray(freq, dtype=np.uint16)
    cap = 4 + 4 * sym.size + 8
    out = np.zeros(cap, dtype=np.uint8)
    fn = lib().eqo_encode_chunk_pairg if grouped else lib().eqo_encode_chunk_pair
    n = fn(_p(sym), sym.size, _p(freq), _p(pt.rank_code), pt.K, _p(pt.pf), pt.fesc, _p(out), cap)
    if n == -2:
        raise ValueError("unknown-symbol")
    if n < 0:
        raise ValueError("buffer")
    return out[:n].tobytes()


def decode_chunk_pair(data: bytes, freq: np.ndarray, pt: PairTable, n: int, grouped: bool = False) -> np.ndarray:
    buf = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    out = np.zeros(max(n, 1), dtype=np.uint8)
    fn = lib().eqo_decode_chunk_pairg if grouped else lib().eqo_decode_chunk_pair
    st = fn(_p(buf), len(data), _p(np.ascontiguousarray(freq, dtype=np.uint16)), _p(pt.rank_code), pt.K, _p(pt.pf),
            pt.fesc, _p(out), n)
    if st == 1:
        raise ValueError("corrupt")
    if st == 2:
        raise ValueError("truncated")
    return out[:n]


def crc32(data) -> int:
    """CRC-32/IEEE of a byte string (the checksum of the uncompressed block
    stream; reflected polynomial 0xEDB88320, init and final XOR 0xFFFFFFFF) — the library routine
    (zlib) as the oracle's one step."""
    import zlib
    return zlib.crc32(bytes(np.ascontiguousarray(data, dtype=np.uint8).reshape(-1))) & 0xFFFFFFFF


# ---------------------------------------------------------------- block (Alg. 1 / Alg. 2)
@dataclass
class OracleBlock:
    layer_shapes: list
    scales: list                     # per layer, uint16 bf16 bits
    freq: np.ndarray                 # uint16[256]
    hist: np.ndarray                 # uint64[256]
    payload: bytes
    chunk_off: np.ndarray            # uint32[n_chunks+1]
    chunk_symbols: int = CHUNK_SYMBOLS
    codes: np.ndarray = field(default=None, repr=False)   # vec(W_q) of the layers, concatenated (layer order)
    fmt: int = FMT_E4M3
    codec: int = CODEC_BYTE
    pair: object = None              # PairTable (codecs CODEC_PAIR, CODEC_PAIR_G)
    chunk_mode: int = CHUNK_LAYER

    @property
    def n_params(self) -> int:
        return int(sum(r * c for r, c in self.layer_shapes))

    @property
    def n_chunks(self) -> int:
        return int(self.chunk_off.size - 1)

    def effective_bits(self) -> float:
        """S:413-417 / SURVEY §8c.12: 8·(payload + offsets + scales + table)/params."""
        rows = sum(r for r, _ in self.layer_shapes)
        b = len(self.payload) + 4 * (self.n_chunks + 1) + 2 * rows + 2 * 256
        return 8.0 * b / self.n_params


def interleave_order(size: int, cs: int) -> np.ndarray:
    """R17: the layer positions in chunk order under CHUNK_INTERLEAVED.  A layer
    of `size` symbols is cut into super-chunks of 32·cs symbols; chunk j (0 ≤ j < 32) of a
    super-chunk holds its 16-symbol groups j, j + 32, j + 64, … (cs / 16 groups), so symbol i
    of that chunk is layer symbol  s·32·cs + (⌊i/16⌋·32 + j)·16 + i mod 16.  The symbols after
    the last whole super-chunk form plain contiguous chunks of cs (the last one ragged), as
    under CHUNK_LAYER.  Returns src with src[q] = the layer position of the q-th symbol in chunk
    order (chunk k is src[k·cs : k·cs + n_k]).  The four nested loops of that definition as one
    broadcast (a loop transcription is checked against it in tests/test_oracle_codec.py)."""
    if cs % IL_GROUP:
        raise ValueError("CHUNK_INTERLEAVED needs chunk_symbols % 16 == 0")
    sc = IL_WAYS * cs
    full = size // sc
    s = np.arange(full, dtype=np.int64)[:, None, None, None]            # super-chunk
    j = np.arange(IL_WAYS, dtype=np.int64)[None, :, None, None]         # chunk within it
    g = np.arange(cs // IL_GROUP, dtype=np.int64)[None, None, :, None]  # group within the chunk
    r = np.arange(IL_GROUP, dtype=np.int64)[None, None, None, :]        # symbol within the group
    head = (s * sc + (g * IL_WAYS + j) * IL_GROUP + r).reshape(-1)      # loop order s, j, g, r
    return np.concatenate([head, np.arange(full * sc, size, dtype=np.int64)])


def segment_sizes(layer_shapes, chunk_mode: int = CHUNK_LAYER) -> np.ndarray:
    """Lengths of the stream segments at whose starts chunking restarts: one per layer
    (CHUNK_LAYER), or one per row (CHUNK_ROW: every row of a layer with K
    columns is split into ⌈K/cs⌉ chunks, e.g. 4096 + 4096 + 4096 + 2048 for K = 14336, so a
    row's chunks are independent K slices of the fused GEMM, §8(f) row 1)."""
    if chunk_mode in (CHUNK_LAYER, CHUNK_INTERLEAVED):
        return np.array([r * c for r, c in layer_shapes], dtype=np.int64)
    if chunk_mode == CHUNK_ROW:
        return np.concatenate([np.full(r, c, dtype=np.int64) for r, c in layer_shapes])
    raise ValueError("chunk_mode")


def encode_codes(codes_list, layer_shapes, scales, cs: int = CHUNK_SYMBOLS, fmt: int = FMT_E4M3,
                 codec: int = CODEC_BYTE, chunk_mode: int = CHUNK_LAYER) -> OracleBlock:
    """Alg. 1 l.4-5 + App. A.1: concatenate vec(W_q) of the block's layers, one table,
    chunked rANS (chunks restart at every segment of ``segment_sizes``)."""
    codes = np.concatenate([np.ascontiguousarray(c, dtype=np.uint8).reshape(-1) for c in codes_list])
    stream = codes
    if chunk_mode == CHUNK_INTERLEAVED:          # the layers' symbols in chunk order (R17)
        for (r, c) in layer_shapes:
            if c % IL_GROUP:
                raise ValueError("CHUNK_INTERLEAVED needs cols % 16 == 0")
        stream = np.concatenate([np.ascontiguousarray(c, dtype=np.uint8).reshape(-1)[interleave_order(c.size, cs)]
                                 for c in codes_list])
    hist = histogram(stream)
    freq = normalize(hist)
    sizes = segment_sizes(layer_shapes, chunk_mode)
    n_chunks = lib().eqo_block_chunks(_p(sizes), sizes.size, cs)
    cap = 4 * n_chunks + 2 * stream.size + 64
    payload = np.zeros(cap, dtype=np.uint8)
    off = np.zeros(n_chunks + 1, dtype=np.uint32)
    pt = None
    if codec in PAIR_CODECS:
        pt = pair_table(hist)
        cap = 4 * n_chunks + 4 * stream.size + 64
        payload = np.zeros(cap, dtype=np.uint8)
        n = lib().eqo_encode_block_pairx(_p(stream), _p(sizes), sizes.size, cs, _p(freq), _p(pt.rank_code),
                                         pt.K, _p(pt.pf), pt.fesc, _p(payload), cap, _p(off), int(codec == CODEC_PAIR_G))
    else:
        n = lib().eqo_encode_block_codec(codec, _p(stream), _p(sizes), sizes.size, cs, _p(freq), _p(payload),
                                         cap, _p(off))
    if n < 0:
        raise ValueError("encode failed %d" % n)
    return OracleBlock(list(layer_shapes), [np.asarray(s, dtype=np.uint16) for s in scales], freq, hist,
                       payload[:n].tobytes(), off, cs, codes, fmt, codec, pt, chunk_mode)


def quantize_encode(layers, lam: float | None = None, scales=None, oct_lo: int = -1, oct_hi: int = 20,
                    cs: int = CHUNK_SYMBOLS, fmt: int = FMT_E4M3, exclude=(), codec: int = CODEC_BYTE,
                    chunk_mode: int = CHUNK_LAYER) -> OracleBlock:
    """Alg. 1 for one block.  ``layers``: list of bf16 [M,N] arrays (uint16 bits or torch).
    Either ``scales`` (per layer) is given, or ``lam`` selects the exhaustive search
    (lam=None -> AbsMax scales, i.e. the λ=0 lossless-FP8 baseline of P:257).  Layers whose
    index is in ``exclude`` keep AbsMax scales (super-weight exclusion)."""
    Ws = [_u16(W) for W in layers]
    shapes = [tuple(W.shape) for W in Ws]
    if scales is None:
        scales = []
        for i, W in enumerate(Ws):
            if lam is None or i in exclude:
                scales.append(absmax_scales(W, fmt))
            else:
                scales.append(search(W, lam, oct_lo, oct_hi, fmt=fmt)[0])
    codes = [quantize(W, S, fmt) for W, S in zip(Ws, scales)]
    return encode_codes(codes, shapes, scales, cs, fmt, codec, chunk_mode)


def decode_block(blk: OracleBlock) -> np.ndarray:
    """Alg. 2 l.1: concatenated symbol stream."""
    sizes = segment_sizes(blk.layer_shapes, blk.chunk_mode)
    out = np.zeros(int(sizes.sum()), dtype=np.uint8)
    payload = np.frombuffer(blk.payload, dtype=np.uint8).copy()
    off = np.ascontiguousarray(blk.chunk_off, dtype=np.uint32)
    if blk.codec in PAIR_CODECS:
        pt = blk.pair
        st = lib().eqo_decode_block_pairx(_p(payload), _p(off), _p(sizes), sizes.size, blk.chunk_symbols,
                                          _p(blk.freq), _p(pt.rank_code), pt.K, _p(pt.pf), pt.fesc, _p(out),
                                          int(blk.codec == CODEC_PAIR_G))
    else:
        st = lib().eqo_decode_block_codec(blk.codec, _p(payload), _p(off), _p(sizes), sizes.size,
                                          blk.chunk_symbols, _p(blk.freq), _p(out))
    if st:
        raise ValueError({1: "corrupt", 2: "truncated"}[st])
    if blk.chunk_mode == CHUNK_INTERLEAVED:      # back from chunk order to layer order (R17)
        res, a = np.empty_like(out), 0
        for (r, c) in blk.layer_shapes:
            res[a + interleave_order(r * c, blk.chunk_symbols)] = out[a:a + r * c]
            a += r * c
        out = res
    return out


def decode_dequant(blk: OracleBlock) -> list:
    """Alg. 2 l.1-2: per-layer bf16 bits of the dequantised weights."""
    stream = decode_block(blk)
    outs, a = [], 0
    for (r, c), S in zip(blk.layer_shapes, blk.scales):
        outs.append(dequant(stream[a:a + r * c].reshape(r, c), S, blk.fmt))
        a += r * c
    return outs


def chunk_table(layer_shapes, cs: int = CHUNK_SYMBOLS, chunk_mode: int = CHUNK_LAYER):
    """(sym0, n) per chunk of a block stream (chunks restart at every segment)."""
    sym0, ns, base = [], [], 0
    for n in segment_sizes(layer_shapes, chunk_mode).tolist():
        for a in range(0, n, cs):
            sym0.append(base + a)
            ns.append(min(cs, n - a))
        base += n
    return np.array(sym0, dtype=np.uint64), np.array(ns, dtype=np.uint32)


def decode_chunks_mt(payload: np.ndarray, chunk_off: np.ndarray, sym0: np.ndarray, ns: np.ndarray,
                     freq: np.ndarray, out: np.ndarray, threads: int, codec: int = CODEC_BYTE) -> None:
    """Multi-threaded oracle decode of selected chunks (CPU baseline timing only)."""
    st = lib().eqo_decode_chunks_mt_codec(codec, _p(payload), _p(chunk_off), _p(sym0), _p(ns), ns.size,
                                    _p(np.ascontiguousarray(freq, dtype=np.uint16)), _p(out), threads)
    if st:
        raise ValueError({1: "corrupt", 2: "truncated"}[st])


def decode_dequant_layer_mt(payload: np.ndarray, chunk_off: np.ndarray, cs: int, rows: int, cols: int,
                            scales: np.ndarray, freq: np.ndarray, threads: int, codec: int = CODEC_BYTE,
                            pair: PairTable | None = None, chunk_mode: int = CHUNK_LAYER) -> np.ndarray:
    """Alg. 2 l.1-2 for one layer's chunks on ``threads`` host threads (CPU baseline)."""
    if chunk_mode == CHUNK_INTERLEAVED:
        # decode in chunk order with one "row" per 16-symbol group (its row's scale), then put
        # every symbol back at its layer position (R17)
        src = interleave_order(rows * cols, cs)
        gscale = np.asarray(scales, dtype=np.uint16)[src[::IL_GROUP] // cols]
        flat = decode_dequant_layer_mt(payload, chunk_off, cs, rows * cols // IL_GROUP, IL_GROUP, gscale, freq,
                                       threads, codec, pair, CHUNK_LAYER).reshape(-1)
        out = np.empty(rows * cols, dtype=np.uint16)
        out[src] = flat
        return out.reshape(rows, cols)
    seg = rows * cols if chunk_mode == CHUNK_LAYER else cols
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    off = np.ascontiguousarray(chunk_off, dtype=np.uint32)
    out = np.zeros(rows * cols, dtype=np.uint16)
    if codec in PAIR_CODECS:
        st = lib().eqo_decode_dequant_layer_mt_pairx_seg(_p(payload), _p(off), off.size - 1, cs, rows * cols, cols,
                                                         seg, _p(np.ascontiguousarray(scales, dtype=np.uint16)),
                                                         _p(np.ascontiguousarray(freq, dtype=np.uint16)),
                                                         _p(pair.rank_code), pair.K, _p(pair.pf), pair.fesc, _p(out),
                                                         threads, int(codec == CODEC_PAIR_G))
        if st:
            raise ValueError({1: "corrupt", 2: "truncated"}[st])
        return out.reshape(rows, cols)
    st = lib().eqo_decode_dequant_layer_mt_codec_seg(codec, _p(payload), _p(off), off.size - 1, cs, rows * cols, cols,
                                                     seg,
                                           _p(np.ascontiguousarray(scales, dtype=np.uint16)),
                                           _p(np.ascontiguousarray(freq, dtype=np.uint16)), _p(out), threads)
    if st:
        raise ValueError({1: "corrupt", 2: "truncated"}[st])
    return out.reshape(rows, cols)
