"""B200-native EntQuant hot path — thin Python binding over libentquant.so (include/entquant.h).

Argument marshalling only: every step of the method runs in the CUDA kernels behind the
C ABI.  PyTorch supplies device memory and streams.  There is no CPU fallback: importing
works without a GPU (for the ABI/export tests), but every compute call requires the
in-tree ``libentquant.so`` and a CUDA device and raises otherwise.

Paper: arXiv 2601.22787 (EntQuant).  Alg. 1 = ``quantize_encode``;
Alg. 2 l.1-2 = ``decode_dequant``.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# EQ_LIB selects an alternative in-tree build (used only for A/B kernel experiments)
LIB_PATH = os.environ.get("EQ_LIB") or os.path.join(_HERE, "libentquant.so")

EQ_OK, EQ_ERR_ARG, EQ_ERR_SHAPE, EQ_ERR_EMPTY, EQ_ERR_BUFFER = 0, 1, 2, 3, 4
EQ_ERR_CORRUPT, EQ_ERR_TRUNCATED, EQ_ERR_UNKNOWN_SYMBOL, EQ_ERR_UNREACHABLE_TARGET, EQ_ERR_CUDA = 5, 6, 7, 8, 9
EQ_FMT_E4M3, EQ_FMT_INT8 = 0, 1
EQ_CODEC_BYTE, EQ_CODEC_WORD, EQ_CODEC_PAIR, EQ_CODEC_PAIR_G = 0, 1, 2, 3
PAIR_CODECS = (EQ_CODEC_PAIR, EQ_CODEC_PAIR_G)   # R15 and its group-ordered form R18: one table layout
# The binding's default codec: the pair codec (R15), the fastest decoder and the lowest rate.
# The C ABI's zero-initialised eq_params keep SPEC's byte codec (R9); pass codec= for it here.
EQ_DEFAULT_CODEC = EQ_CODEC_PAIR_G
EQ_OUT_FP8, EQ_OUT_BF16 = 0, 1
EQ_CHUNK_LAYER, EQ_CHUNK_ROW, EQ_CHUNK_INTERLEAVED = 0, 1, 2
EQ_SCALES_SEARCH, EQ_SCALES_ABSMAX, EQ_SCALES_GIVEN = 0, 1, 2
EQ_MAX_LAYERS = 8
EQ_DEFAULT_CHUNK = 4096
EQ_PROB_BITS = 12
EQ_PAYLOAD_SLACK = 256
EQ_ARENA_ALIGN = 256

EXPORTS = (
    "eq_status_string", "eq_version", "eq_encode_bounds", "eq_arena_layout", "eq_absmax",
    "eq_search_scratch_bytes", "eq_search_scales", "eq_quantize_hist", "eq_build_table", "eq_build_pair_table",
    "eq_decode_lanes",
    "eq_rans_encode", "eq_quantize_encode", "eq_decode_dequant", "eq_decode_host_workspace_bytes",
    "eq_decode_dequant_host", "eq_check", "eq_calibrate_scratch_bytes", "eq_calibrate_lambda",
    "eq_qmatmul",
    "eq_qmatmul_group",
    "eq_qmatmul_workspace_bytes",
    "eq_lbfgs_default_params",
    "eq_lbfgs_scratch_bytes",
    "eq_lbfgs_scales",
    "eq_rd_eval",
    "eq_crc32_scratch_bytes",
    "eq_crc32",
)


class EqError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} ({status})")


class eq_tensor(ctypes.Structure):
    _fields_ = [("w", ctypes.c_void_p), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64)]


class eq_params(ctypes.Structure):
    _fields_ = [("format", ctypes.c_uint32), ("chunk_symbols", ctypes.c_uint32),
                ("prob_bits", ctypes.c_uint32), ("scale_mode", ctypes.c_uint32),
                ("lambda_", ctypes.c_double), ("oct_lo", ctypes.c_int32), ("oct_hi", ctypes.c_int32),
                ("exclude_mask", ctypes.c_uint32), ("codec", ctypes.c_uint32), ("chunk_mode", ctypes.c_uint32)]


class eq_lbfgs_params(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_uint32), ("history", ctypes.c_uint32), ("trials", ctypes.c_uint32),
                ("max_backtracks", ctypes.c_uint32), ("lr", ctypes.c_double), ("c1", ctypes.c_double),
                ("grad_tol", ctypes.c_double), ("change_tol", ctypes.c_double)]


class eq_block(ctypes.Structure):
    _fields_ = [("payload", ctypes.c_void_p), ("payload_cap", ctypes.c_uint64),
                ("payload_bytes", ctypes.c_uint64), ("chunk_off", ctypes.c_void_p),
                ("n_chunks", ctypes.c_uint32), ("chunk_symbols", ctypes.c_uint32),
                ("freq", ctypes.c_void_p), ("scales", ctypes.c_void_p), ("n_layers", ctypes.c_uint32),
                ("format", ctypes.c_uint32),
                ("layer_rows", ctypes.c_int64 * EQ_MAX_LAYERS), ("layer_cols", ctypes.c_int64 * EQ_MAX_LAYERS),
                ("codec", ctypes.c_uint32), ("chunk_mode", ctypes.c_uint32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Loads the in-tree library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libentquant.so missing at {LIB_PATH}: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P, u32, u64, i32, dbl = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double
        st = ctypes.c_int
        sig = {
            "eq_status_string": (ctypes.c_char_p, [st]),
            "eq_version": (ctypes.c_char_p, []),
            "eq_encode_bounds": (st, [P, u32, P, P, P, P]),
            "eq_arena_layout": (st, [P, u32, u32, P, P]),
            "eq_absmax": (st, [P, u32, P, P]),
            "eq_search_scratch_bytes": (u64, [P]),
            "eq_search_scales": (st, [P, u32, P, u32, i32, i32, P, u32, P, P, P, u64, P]),
            "eq_quantize_hist": (st, [P, u32, P, P, u32, P, P, P]),
            "eq_build_table": (st, [P, P, P, P]),
            "eq_build_pair_table": (st, [P, P, P, P]),
            "eq_decode_lanes": (st, [u32, u32, ctypes.c_int, P]),
            "eq_rans_encode": (st, [P, P, P, P, P, P]),
            "eq_quantize_encode": (st, [P, u32, P, P, P, u64, P]),
            "eq_decode_dequant": (st, [P, u32, u32, P, u64, P, P]),
            "eq_decode_host_workspace_bytes": (u64, [P, u32, u32]),
            "eq_decode_dequant_host": (st, [P, u32, u32, P, u64, P, u64, P]),
            "eq_check": (st, [P, P]),
            "eq_calibrate_scratch_bytes": (u64, [P, u32, u32]),
            "eq_calibrate_lambda": (st, [P, u32, P, dbl, u32, P, P, P, u64, P]),
            "eq_qmatmul": (st, [P, u32, P, u32, P, P, u64, P, P]),
            "eq_qmatmul_group": (st, [P, u32, P, P, P, u32, P, u64, P, P]),
            "eq_qmatmul_workspace_bytes": (u64, [P, u32, P, u32]),
            "eq_lbfgs_default_params": (None, [P]),
            "eq_lbfgs_scratch_bytes": (u64, [P, u32, P]),
            "eq_lbfgs_scales": (st, [P, u32, u32, dbl, P, P, P, P, P, u64, P]),
            "eq_rd_eval": (st, [P, u32, dbl, P, P, P, P, u64, P]),
            "eq_crc32_scratch_bytes": (u64, [u64]),
            "eq_crc32": (st, [P, u64, P, P, u64, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().eq_status_string(s).decode()


def version() -> str:
    return lib().eq_version().decode()


def _ck(status: int, where: str) -> None:
    if status != EQ_OK:
        raise EqError(status, where)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _require_cuda(*ts) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("entquant: tensors must be CUDA tensors (no CPU fallback)")


def _tensor(W: torch.Tensor) -> eq_tensor:
    if W.dtype != torch.bfloat16 or W.dim() != 2 or not W.is_contiguous():
        raise ValueError("weights must be contiguous 2-D bf16")
    _require_cuda(W)
    return eq_tensor(W.data_ptr(), W.shape[0], W.shape[1])


def _params(chunk_symbols=EQ_DEFAULT_CHUNK, scale_mode=EQ_SCALES_SEARCH, lam=0.0, oct_lo=-1, oct_hi=20,
            fmt=EQ_FMT_E4M3, exclude=(), codec=EQ_CODEC_BYTE, chunk_mode=EQ_CHUNK_LAYER) -> eq_params:
    mask = 0
    for i in exclude:
        mask |= 1 << int(i)
    return eq_params(fmt, chunk_symbols, EQ_PROB_BITS, scale_mode, float(lam), oct_lo, oct_hi, mask, codec, chunk_mode)


# ---------------------------------------------------------------- compressed block
@dataclass
class Block:
    """One compressed transformer block (z, S*, ℳ of Alg. 1) held in device memory."""
    payload: torch.Tensor            # uint8 [payload_cap]
    payload_bytes: int
    chunk_off: torch.Tensor          # int32 (uint32 bits) [n_chunks+1]
    freq: torch.Tensor               # int16 (uint16 bits) [256]
    scales: torch.Tensor             # bf16 [Σ rows]
    shapes: list                     # [(rows, cols)] in block order
    chunk_symbols: int = EQ_DEFAULT_CHUNK
    meta: dict = field(default_factory=dict)
    format: int = EQ_FMT_E4M3
    codec: int = EQ_CODEC_BYTE
    chunk_mode: int = EQ_CHUNK_LAYER
    crc: int | None = None           # CRC-32 of the block's codes at encode time (verify mode)

    @property
    def n_chunks(self) -> int:
        return self.chunk_off.numel() - 1

    @property
    def n_params(self) -> int:
        return sum(r * c for r, c in self.shapes)

    def c_struct(self) -> eq_block:
        b = eq_block()
        b.payload = self.payload.data_ptr()
        b.payload_cap = self.payload.numel()
        b.payload_bytes = self.payload_bytes
        b.chunk_off = self.chunk_off.data_ptr()
        b.n_chunks = self.n_chunks
        b.chunk_symbols = self.chunk_symbols
        b.freq = self.freq.data_ptr()
        b.scales = self.scales.data_ptr()
        b.n_layers = len(self.shapes)
        b.format = self.format
        b.codec = self.codec
        b.chunk_mode = self.chunk_mode
        for i, (r, c) in enumerate(self.shapes):
            b.layer_rows[i] = r
            b.layer_cols[i] = c
        return b

    def compressed_bytes(self) -> int:
        """payload + chunk offsets + bf16 scales + table: 256×u16, 512×u16 with the pair table
        (S:413-417)."""
        rows = sum(r for r, _ in self.shapes)
        return self.payload_bytes + 4 * (self.n_chunks + 1) + 2 * rows + 2 * self.freq.numel()

    def effective_bits(self) -> float:
        return 8.0 * self.compressed_bytes() / self.n_params

    def decode_read_bytes(self) -> int:
        """Algorithmic bytes a decode reads: payload + offsets + scales + table."""
        return self.compressed_bytes()


def encode_bounds(layers, chunk_symbols=EQ_DEFAULT_CHUNK, codec: int = EQ_DEFAULT_CODEC, chunk_mode: int = EQ_CHUNK_LAYER):
    ts = (eq_tensor * len(layers))(*[eq_tensor(0 if not W.is_cuda else W.data_ptr(), W.shape[0], W.shape[1]) for W in layers])
    for i, W in enumerate(layers):
        ts[i].w = 1 if ts[i].w == 0 else ts[i].w       # sizing does not dereference
    p = _params(chunk_symbols, codec=codec, chunk_mode=chunk_mode)
    cap, nc, sb = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint64()
    _ck(lib().eq_encode_bounds(ts, len(layers), ctypes.byref(p), ctypes.byref(cap), ctypes.byref(nc), ctypes.byref(sb)),
        "eq_encode_bounds")
    return cap.value, nc.value, sb.value


def quantize_encode(layers, lam: float = 0.0, scale_mode: int = EQ_SCALES_SEARCH, scales: torch.Tensor | None = None,
                    chunk_symbols: int = EQ_DEFAULT_CHUNK, oct_lo: int = -1, oct_hi: int = 20,
                    stream=None, scratch: torch.Tensor | None = None, shrink: bool = True,
                    format: int = EQ_FMT_E4M3, exclude=(), codec: int = EQ_DEFAULT_CODEC,
                    chunk_mode: int = EQ_CHUNK_LAYER, crc: bool = False) -> Block:
    """Alg. 1 for one block of bf16 CUDA matrices.  Synchronous (reads payload size).
    ``crc``: also record the CRC-32 of the block's codes (the verify mode, ``verify_crc``).
    ``exclude``: layer indices kept at AbsMax scales (λ = 0); ``codec``: rANS
    renormalisation (EQ_CODEC_BYTE, R9 / EQ_CODEC_WORD, R14 / EQ_CODEC_PAIR, R15 / EQ_CODEC_PAIR_G, R18);
    ``chunk_mode``: EQ_CHUNK_LAYER, EQ_CHUNK_ROW (chunks also restart at row starts) or
    EQ_CHUNK_INTERLEAVED (R17: 16-symbol groups dealt to 32 chunks in turn; pair codec)."""
    if scales is not None:
        scale_mode = EQ_SCALES_GIVEN
    dev = layers[0].device
    ts = (eq_tensor * len(layers))(*[_tensor(W) for W in layers])
    p = _params(chunk_symbols, scale_mode, lam, oct_lo, oct_hi, format, exclude, codec, chunk_mode)
    cap, nc, sb = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint64()
    _ck(lib().eq_encode_bounds(ts, len(layers), ctypes.byref(p), ctypes.byref(cap), ctypes.byref(nc), ctypes.byref(sb)),
        "eq_encode_bounds")
    rows = sum(W.shape[0] for W in layers)
    payload = torch.empty(cap.value, dtype=torch.uint8, device=dev)
    off = torch.empty(nc.value + 1, dtype=torch.int32, device=dev)
    freq = torch.zeros(512 if codec in PAIR_CODECS else 256, dtype=torch.int16, device=dev)
    if scales is None:
        scales = torch.empty(rows, dtype=torch.bfloat16, device=dev)
    else:
        _require_cuda(scales)
        scales = scales.contiguous()
    if scratch is None or scratch.numel() < sb.value:
        scratch = torch.empty(sb.value, dtype=torch.uint8, device=dev)
    b = eq_block()
    b.payload, b.payload_cap = payload.data_ptr(), cap.value
    b.chunk_off, b.freq, b.scales = off.data_ptr(), freq.data_ptr(), scales.data_ptr()
    _ck(lib().eq_quantize_encode(ts, len(layers), ctypes.byref(p), ctypes.byref(b), scratch.data_ptr(), scratch.numel(),
                                 _stream(stream)), "eq_quantize_encode")
    nbytes = b.payload_bytes
    crc_val = None
    if crc:      # the codes stream sits at the start of the scratch (include/entquant.h, eq_crc32)
        crc_val = crc32(scratch[:sum(W.numel() for W in layers)], stream)
    if shrink:   # keep only what the block needs (+ decoder read slack)
        keep = (nbytes + EQ_PAYLOAD_SLACK + 255) // 256 * 256
        payload = payload[:keep].clone()
    return Block(payload, nbytes, off, freq, scales, [tuple(W.shape) for W in layers], chunk_symbols,
                 {"lambda": lam, "scale_mode": scale_mode, "exclude": tuple(exclude)}, format, codec, chunk_mode,
                 crc_val)


def crc32(data: torch.Tensor, stream=None) -> int:
    """CRC-32/IEEE of a CUDA byte tensor, computed on the GPU (eq_crc32).  Synchronous."""
    _require_cuda(data)
    data = data.contiguous().view(torch.uint8).reshape(-1)
    n = data.numel()
    scratch = torch.empty(max(1, lib().eq_crc32_scratch_bytes(n)), dtype=torch.uint8, device=data.device)
    out = torch.empty(1, dtype=torch.int32, device=data.device)
    _ck(lib().eq_crc32(data.data_ptr() if n else None, n, out.data_ptr(), scratch.data_ptr(), scratch.numel(),
                       _stream(stream)), "eq_crc32")
    return int(out.item()) & 0xFFFFFFFF


def verify_crc(blocks, stream=None) -> list:
    """The verify mode: decode the blocks to their codes (EQ_OUT_FP8),
    CRC-32 each block's layers in order and compare with the CRC recorded at encode time.
    Returns the per-block verdicts (True = match); raises EqError on a stream error."""
    dec = Decoder(blocks, EQ_OUT_FP8)
    dec(stream)
    dec.check(stream)
    ok = []
    for b, vs in zip(blocks, dec.views()):
        if b.crc is None:
            raise ValueError("block encoded without crc=True")
        codes = torch.cat([v.reshape(-1).view(torch.uint8) for v in vs])
        ok.append(crc32(codes, stream) == b.crc)
    return ok


def arena_layout(blocks, out_dtype=EQ_OUT_BF16):
    arr = (eq_block * len(blocks))(*[b.c_struct() for b in blocks])
    offs = (ctypes.c_uint64 * (EQ_MAX_LAYERS * len(blocks)))()
    total = ctypes.c_uint64()
    _ck(lib().eq_arena_layout(arr, len(blocks), out_dtype, offs, ctypes.byref(total)), "eq_arena_layout")
    return [list(offs[b * EQ_MAX_LAYERS:(b + 1) * EQ_MAX_LAYERS]) for b in range(len(blocks))], total.value


class Decoder:
    """Pre-marshalled decode of a fixed list of blocks into one arena (Alg. 2 l.1-2, App. A.1):
    builds the C descriptors once; ``__call__`` is one eq_decode_dequant call."""

    def __init__(self, blocks, out_dtype=EQ_OUT_BF16, arena: torch.Tensor | None = None):
        self.blocks = list(blocks)
        self.out_dtype = out_dtype
        self.offsets, self.total = arena_layout(self.blocks, out_dtype)
        dev = self.blocks[0].payload.device
        if arena is None:
            arena = torch.empty(self.total, dtype=torch.uint8, device=dev)
        if arena.numel() < self.total:
            raise EqError(EQ_ERR_BUFFER, "Decoder arena")
        self.arena = arena
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self._arr = (eq_block * len(self.blocks))(*[b.c_struct() for b in self.blocks])

    def __call__(self, stream=None) -> None:
        _ck(lib().eq_decode_dequant(self._arr, len(self.blocks), self.out_dtype, self.arena.data_ptr(),
                                    self.arena.numel(), self.err.data_ptr(), _stream(stream)), "eq_decode_dequant")

    def check(self, stream=None) -> None:
        _ck(lib().eq_check(self.err.data_ptr(), _stream(stream)), "eq_check")

    def views(self):
        """Per block, per layer tensor views into the arena (no copies)."""
        dt = torch.bfloat16 if self.out_dtype == EQ_OUT_BF16 else torch.float8_e4m3fn
        es = 2 if self.out_dtype == EQ_OUT_BF16 else 1
        out = []
        for b, offs in zip(self.blocks, self.offsets):
            vs = []
            for (r, c), o in zip(b.shapes, offs):
                vs.append(self.arena[o:o + r * c * es].view(dt).view(r, c))
            out.append(vs)
        return out


def decode_lanes(codec: int = EQ_CODEC_PAIR, out_dtype: int = EQ_OUT_BF16, device: int | None = None) -> int:
    """Chunks the decoder keeps in flight at once on a device (one chunk per lane)."""
    if device is None:
        device = torch.cuda.current_device()
    n = ctypes.c_uint64()
    _ck(lib().eq_decode_lanes(codec, out_dtype, device, ctypes.byref(n)), "eq_decode_lanes")
    return int(n.value)


def decode_dequant(blocks, out_dtype=EQ_OUT_BF16, stream=None, check: bool = True):
    """Decodes blocks (one launch) and returns per-block lists of per-layer views."""
    d = Decoder(blocks, out_dtype)
    d(stream)
    if check:
        d.check(stream)
    return d.views()


class HostBlocks:
    """Pinned host copies of blocks for the end-to-end (host buffer) decode."""

    def __init__(self, blocks, out_dtype=EQ_OUT_BF16):
        self.blocks = list(blocks)
        self.out_dtype = out_dtype
        self.host = []
        for b in self.blocks:
            h = {
                "payload": b.payload[:b.payload_bytes + EQ_PAYLOAD_SLACK].cpu().pin_memory(),
                "off": b.chunk_off.cpu().pin_memory(),
                "freq": b.freq.cpu().pin_memory(),
                "scales": b.scales.cpu().pin_memory(),
            }
            self.host.append(h)
        self._arr = (eq_block * len(self.blocks))()
        for i, (b, h) in enumerate(zip(self.blocks, self.host)):
            s = b.c_struct()
            s.payload, s.payload_cap = h["payload"].data_ptr(), h["payload"].numel()
            s.chunk_off, s.freq, s.scales = h["off"].data_ptr(), h["freq"].data_ptr(), h["scales"].data_ptr()
            self._arr[i] = s
        self.ws_bytes = lib().eq_decode_host_workspace_bytes(self._arr, len(self.blocks), out_dtype)
        _, self.total = arena_layout(self.blocks, out_dtype)
        self.arena_host = torch.empty(self.total, dtype=torch.uint8).pin_memory()
        self.workspace = None

    def h2d_bytes(self) -> int:
        """Bytes copied host->device per decode: payload + offsets + table + scales."""
        return sum(b.payload_bytes + 4 * (b.n_chunks + 1) + 2 * b.freq.numel() + 2 * b.scales.numel() for b in self.blocks)

    def decode(self, stream=None) -> torch.Tensor:
        if self.workspace is None:
            self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.blocks[0].payload.device)
        _ck(lib().eq_decode_dequant_host(self._arr, len(self.blocks), self.out_dtype, self.arena_host.data_ptr(),
                                         self.arena_host.numel(), self.workspace.data_ptr(), self.workspace.numel(),
                                         _stream(stream)), "eq_decode_dequant_host")
        return self.arena_host


# ---------------------------------------------------------------- step-level calls (a1-a6)
def absmax(W: torch.Tensor, stream=None, format: int = EQ_FMT_E4M3) -> torch.Tensor:
    t = _tensor(W)
    s0 = torch.empty(W.shape[0], dtype=torch.bfloat16, device=W.device)
    _ck(lib().eq_absmax(ctypes.byref(t), format, s0.data_ptr(), _stream(stream)), "eq_absmax")
    return s0


def search_scales(W: torch.Tensor, lambdas, oct_lo: int = -1, oct_hi: int = 20, rows: torch.Tensor | None = None,
                  with_obj: bool = False, stream=None, format: int = EQ_FMT_E4M3):
    """a2: scales [len(lambdas), rows] (bf16) and optionally the per-row objective (f64)."""
    t = _tensor(W)
    lam = list(lambdas) if hasattr(lambdas, "__len__") else [float(lambdas)]
    la = (ctypes.c_double * len(lam))(*lam)
    sc = torch.zeros(len(lam), W.shape[0], dtype=torch.bfloat16, device=W.device)
    ob = torch.zeros(len(lam), W.shape[0], dtype=torch.float64, device=W.device) if with_obj else None
    sb = lib().eq_search_scratch_bytes(ctypes.byref(t))
    scratch = torch.empty(sb, dtype=torch.uint8, device=W.device)
    if rows is not None:
        rows = rows.to(device=W.device, dtype=torch.int32).contiguous()
    _ck(lib().eq_search_scales(ctypes.byref(t), format, la, len(lam), oct_lo, oct_hi, _ptr(rows),
                               0 if rows is None else rows.numel(), sc.data_ptr(), _ptr(ob), scratch.data_ptr(), sb,
                               _stream(stream)), "eq_search_scales")
    return (sc, ob) if with_obj else sc


def quantize_hist(W: torch.Tensor, scales: torch.Tensor, codes: bool = True, hist: torch.Tensor | None = None,
                  rows: torch.Tensor | None = None, stream=None, format: int = EQ_FMT_E4M3):
    """a3+a4: (codes uint8 [M,N] or None, hist int64 [256] accumulated)."""
    t = _tensor(W)
    _require_cuda(scales)
    c = torch.empty(W.shape, dtype=torch.uint8, device=W.device) if codes else None
    if hist is None:
        hist = torch.zeros(256, dtype=torch.int64, device=W.device)
    if rows is not None:
        rows = rows.to(device=W.device, dtype=torch.int32).contiguous()
    _ck(lib().eq_quantize_hist(ctypes.byref(t), format, scales.contiguous().data_ptr(), _ptr(rows),
                               0 if rows is None else rows.numel(), _ptr(c), hist.data_ptr(), _stream(stream)),
        "eq_quantize_hist")
    return c, hist


def build_table(hist: torch.Tensor, stream=None):
    """a5: (freq int16 [256], device error word)."""
    _require_cuda(hist)
    freq = torch.empty(256, dtype=torch.int16, device=hist.device)
    err = torch.zeros(1, dtype=torch.int32, device=hist.device)
    _ck(lib().eq_build_table(hist.data_ptr(), freq.data_ptr(), err.data_ptr(), _stream(stream)), "eq_build_table")
    return freq, err


def build_pair_table(hist: torch.Tensor, stream=None):
    """a5 for EQ_CODEC_PAIR (R15): (table int16 [512] — [0,256) the single table of
    build_table, [256,512) the pair table — and the device error word)."""
    _require_cuda(hist)
    tab = torch.zeros(512, dtype=torch.int16, device=hist.device)
    err = torch.zeros(1, dtype=torch.int32, device=hist.device)
    _ck(lib().eq_build_table(hist.data_ptr(), tab.data_ptr(), err.data_ptr(), _stream(stream)), "eq_build_table")
    _ck(lib().eq_build_pair_table(hist.data_ptr(), tab.data_ptr(), err.data_ptr(), _stream(stream)),
        "eq_build_pair_table")
    return tab, err


def rans_encode(codes: torch.Tensor, shapes, freq: torch.Tensor, scales: torch.Tensor | None = None,
                chunk_symbols: int = EQ_DEFAULT_CHUNK, stream=None, codec: int = EQ_DEFAULT_CODEC,
                chunk_mode: int = EQ_CHUNK_LAYER) -> Block:
    """a6 alone: encode a concatenated symbol stream (uint8 CUDA) with a given table."""
    _require_cuda(codes, freq)
    n = sum(r * c for r, c in shapes)
    if chunk_mode == EQ_CHUNK_ROW:
        nc = sum(r * ((c + chunk_symbols - 1) // chunk_symbols) for r, c in shapes)
    else:
        nc = sum((r * c + chunk_symbols - 1) // chunk_symbols for r, c in shapes)
    cap = (4 * nc + (3 if codec in PAIR_CODECS else 2) * n + EQ_PAYLOAD_SLACK + 255) // 256 * 256
    dev = codes.device
    blk = Block(torch.empty(cap, dtype=torch.uint8, device=dev), 0, torch.empty(nc + 1, dtype=torch.int32, device=dev),
                freq, scales if scales is not None else torch.ones(sum(r for r, _ in shapes), dtype=torch.bfloat16, device=dev),
                list(shapes), chunk_symbols, codec=codec, chunk_mode=chunk_mode)
    sizes = torch.empty(max(nc, 1), dtype=torch.int32, device=dev)
    tot = torch.zeros(1, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    s = blk.c_struct()
    _ck(lib().eq_rans_encode(codes.data_ptr(), ctypes.byref(s), sizes.data_ptr(), tot.data_ptr(), err.data_ptr(),
                             _stream(stream)), "eq_rans_encode")
    _ck(lib().eq_check(err.data_ptr(), _stream(stream)), "eq_rans_encode(check)")
    blk.payload_bytes = int(tot.item())
    return blk


def calibrate_lambda(layers, target_bits: float, row_stride: int = 8, chunk_symbols: int = EQ_DEFAULT_CHUNK,
                     oct_lo: int = -1, oct_hi: int = 20, stream=None, format: int = EQ_FMT_E4M3,
                     codec: int = EQ_DEFAULT_CODEC, chunk_mode: int = EQ_CHUNK_LAYER):
    """Global λ for a target effective rate.  Returns (λ, estimated bits);
    ``codec`` sizes the per-block table and ``chunk_mode`` the chunk count in the side information."""
    ts = (eq_tensor * len(layers))(*[_tensor(W) for W in layers])
    p = _params(chunk_symbols, EQ_SCALES_SEARCH, 0.0, oct_lo, oct_hi, format, codec=codec, chunk_mode=chunk_mode)
    sb = lib().eq_calibrate_scratch_bytes(ts, len(layers), row_stride)
    scratch = torch.empty(sb, dtype=torch.uint8, device=layers[0].device)
    lam, est = ctypes.c_double(), ctypes.c_double()
    _ck(lib().eq_calibrate_lambda(ts, len(layers), ctypes.byref(p), float(target_bits), row_stride, ctypes.byref(lam),
                                  ctypes.byref(est), scratch.data_ptr(), sb, _stream(stream)), "eq_calibrate_lambda")
    return lam.value, est.value


def lbfgs_params(**kw) -> eq_lbfgs_params:
    """eq_lbfgs_params with the library defaults, overridden by keyword."""
    p = eq_lbfgs_params()
    lib().eq_lbfgs_default_params(ctypes.byref(p))
    for k, v in kw.items():
        if v is not None:
            setattr(p, k, v)
    return p


def lbfgs_scales(layers, lam: float, format: int = EQ_FMT_E4M3, stream=None, **params):
    """Alg. 1 l.2 by the paper's solver: L-BFGS + STE on each layer's scales.
    Returns (scales bf16 [Σ rows], trace f64 [n_layers, max_iters+1], info int [n_layers, 4])."""
    dev = layers[0].device
    ts = (eq_tensor * len(layers))(*[_tensor(W) for W in layers])
    p = lbfgs_params(**params)
    sb = lib().eq_lbfgs_scratch_bytes(ts, len(layers), ctypes.byref(p))
    if sb == 0:
        raise EqError(EQ_ERR_ARG, "eq_lbfgs_scratch_bytes")
    scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
    R = sum(int(W.shape[0]) for W in layers)
    scales = torch.empty(R, dtype=torch.bfloat16, device=dev)
    trace = torch.empty(len(layers), p.max_iters + 1, dtype=torch.float64, device=dev)
    info = torch.zeros(len(layers), 4, dtype=torch.int32, device=dev)
    _ck(lib().eq_lbfgs_scales(ts, len(layers), format, float(lam), ctypes.byref(p), scales.data_ptr(),
                              trace.data_ptr(), info.data_ptr(), scratch.data_ptr(), sb, _stream(stream)),
        "eq_lbfgs_scales")
    return scales, trace, info


def rd_eval(W: torch.Tensor, scales: torch.Tensor, lam: float, format: int = EQ_FMT_E4M3, stream=None):
    """Eq. 4 at given bf16 scales and its straight-through gradient w.r.t. log2 s:
    (objective f64 [1], gradient f64 [rows])."""
    _require_cuda(W, scales)
    t = _tensor(W)
    sb = lib().eq_lbfgs_scratch_bytes(ctypes.byref(t), 1, None)
    scratch = torch.empty(sb, dtype=torch.uint8, device=W.device)
    f = torch.empty(1, dtype=torch.float64, device=W.device)
    g = torch.empty(W.shape[0], dtype=torch.float64, device=W.device)
    _ck(lib().eq_rd_eval(ctypes.byref(t), format, float(lam), scales.contiguous().data_ptr(), f.data_ptr(),
                         g.data_ptr(), scratch.data_ptr(), sb, _stream(stream)), "eq_rd_eval")
    return f, g


def check(err: torch.Tensor, stream=None) -> None:
    _ck(lib().eq_check(err.data_ptr(), _stream(stream)), "eq_check")


def qmatmul_group(block: Block, layers: list[int], xs: list[torch.Tensor], ys: list[torch.Tensor] | None = None,
                  err: torch.Tensor | None = None, stream=None, check: bool = True,
                  workspace: torch.Tensor | None = None) -> list[torch.Tensor]:
    """Alg. 2 l.3 fused with decoding (NEXT row 1): ys[q] = xs[q] · Ŵ_{layers[q]}ᵀ, fp32
    [batch, rows], for several layers of ``block`` in one launch; weights are decoded
    straight into tcgen05 tiles."""
    if len(layers) != len(xs) or not layers:
        raise ValueError("one x per layer")
    batch = xs[0].shape[0]
    for x, l in zip(xs, layers):
        if x.dtype != torch.bfloat16 or x.dim() != 2 or not x.is_contiguous() or x.shape[0] != batch:
            raise ValueError("xs must be contiguous 2-D bf16 with a common batch")
        _require_cuda(x)
        if not 0 <= l < len(block.shapes) or x.shape[1] != block.shapes[l][1]:
            raise EqError(EQ_ERR_SHAPE, "qmatmul")
    dev = xs[0].device
    if ys is None:
        ys = [torch.empty(batch, block.shapes[l][0], dtype=torch.float32, device=dev) for l in layers]
    own = err is None
    if own:
        err = torch.zeros(1, dtype=torch.int32, device=dev)
    b = block.c_struct()
    n = len(layers)
    la = (ctypes.c_uint32 * n)(*layers)
    xa = (ctypes.c_void_p * n)(*[x.data_ptr() for x in xs])
    ya = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys])
    need = lib().eq_qmatmul_workspace_bytes(ctypes.byref(b), n, la, batch)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
    _ck(lib().eq_qmatmul_group(ctypes.byref(b), n, la, xa, ya, batch, workspace.data_ptr(), workspace.numel(),
                               err.data_ptr(), _stream(stream)), "eq_qmatmul_group")
    if check and own:
        _ck(lib().eq_check(err.data_ptr(), _stream(stream)), "eq_qmatmul(check)")
    return ys


def qmatmul(block: Block, layer: int, x: torch.Tensor, y: torch.Tensor | None = None, err: torch.Tensor | None = None,
            stream=None, check: bool = True, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Single-layer :func:`qmatmul_group`."""
    return qmatmul_group(block, [layer], [x], None if y is None else [y], err, stream, check, workspace)[0]
