"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no quantiser, scale, entropy or codec
step).  It only produces bf16 weight matrices of Llama shapes with heavy-tailed
(Student-t / Gaussian-mixture) entries, the recipe stated in DESIGN.md §5:

    u      = lowbias32(lowbias32(idx ^ k1) + k2)        counter-based 32-bit hash
    t      = Q[u >> 12]                                  2^20-entry fp32 quantile table
    W[i,j] = bf16_rne(fp32(t) * g_i)                     g_i = fp32(σ·exp(0.3·z_i))

Q is the quantile function of the chosen distribution at p = (k+0.5)/2^20, computed once
in float64 on the host; g_i is a per-row log-normal channel spread (z_i a normal quantile
from the row hash).  Only integer ops, a table gather and ONE fp32 multiply + RNE cast
touch the data, so torch produces bit-identical matrices on CPU and CUDA (tested).
"""
from __future__ import annotations

import functools
import hashlib

import numpy as np
import torch

SIGMA = 0.02
ROW_SPREAD = 0.3
TABLE_BITS = 20
_MASK32 = 0xFFFFFFFF

DISTS = ("t4", "t3", "gauss", "mix")

# Llama shapes (HF module order q, k, v, o, gate, up, down; DESIGN.md §3 reading R6).
LLAMA = {
    "llama-3.2-1b": dict(hidden=2048, kv=512, inter=8192, layers=16),
    "llama-3-8b": dict(hidden=4096, kv=1024, inter=14336, layers=32),
    "llama-3-70b": dict(hidden=8192, kv=1024, inter=28672, layers=80),
}
MATRIX_NAMES = ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj")


def block_shapes(model: str):
    """[(rows=out_features, cols=in_features)] of one decoder block's 7 linear layers."""
    c = LLAMA[model]
    h, kv, it = c["hidden"], c["kv"], c["inter"]
    return [(h, h), (kv, h), (kv, h), (h, h), (it, h), (it, h), (h, it)]


def _key(*parts) -> int:
    d = hashlib.sha256(("eqsynth:" + ":".join(str(p) for p in parts)).encode()).digest()
    return int.from_bytes(d[:4], "little")


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for int64 tensors holding uint32 values, without int64 overflow."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _MASK32


def lowbias32(x: torch.Tensor) -> torch.Tensor:
    """C. Wellons' lowbias32 integer hash on uint32 values stored in int64."""
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


@functools.lru_cache(maxsize=None)
def quantile_table(dist: str) -> np.ndarray:
    """fp32 quantiles at p=(k+0.5)/2^20 (float64 closed forms / scipy, rounded once)."""
    from scipy import special, stats
    n = 1 << TABLE_BITS
    p = (np.arange(n, dtype=np.float64) + 0.5) / n
    if dist == "t4":
        q = stats.t.ppf(p, 4)
    elif dist == "t3":
        q = stats.t.ppf(p, 3)
    elif dist == "gauss":
        q = special.ndtri(p)
    elif dist == "mix":
        # 0.98·N(0,1) + 0.02·N(0,8²): the mixture's quantile function by bisection on its CDF
        cdf = lambda x: 0.98 * special.ndtr(x) + 0.02 * special.ndtr(x / 8.0)
        lo, hi = np.full(n, -80.0), np.full(n, 80.0)
        for _ in range(80):
            mid = 0.5 * (lo + hi)
            m = cdf(mid) < p
            lo = np.where(m, mid, lo)
            hi = np.where(m, hi, mid)
        q = 0.5 * (lo + hi)
    else:
        raise ValueError(dist)
    return q.astype(np.float32)


def _table(dist: str, device) -> torch.Tensor:
    return torch.from_numpy(quantile_table(dist)).to(device)


def row_gains(rows: int, seed: int, layer: int, matrix: int, sigma: float = SIGMA) -> np.ndarray:
    """fp32 per-row factors σ·exp(0.3·z_i), z_i = normal quantile of a row hash (host f64)."""
    from scipy import special
    k = _key(seed, layer, matrix, "rows")
    idx = torch.arange(rows, dtype=torch.int64)
    u = lowbias32(lowbias32(idx ^ k) + 0x9E3779B9 & _MASK32).numpy()
    z = special.ndtri(((u >> 12).astype(np.float64) + 0.5) / (1 << TABLE_BITS))
    return (sigma * np.exp(ROW_SPREAD * z)).astype(np.float32)


def weights(rows: int, cols: int, seed: int = 0, layer: int = 0, matrix: int = 0,
            dist: str = "t4", device="cpu", outliers: int = 0) -> torch.Tensor:
    """bf16 [rows, cols] synthetic weight matrix, bit-identical on every device.

    ``outliers`` plants that many ~100σ entries (super-weight-like) at hashed
    positions."""
    device = torch.device(device)
    k1, k2 = _key(seed, layer, matrix, dist, "a"), _key(seed, layer, matrix, dist, "b")
    tab = _table(dist, device)
    gains = torch.from_numpy(row_gains(rows, seed, layer, matrix)).to(device)
    out = torch.empty(rows, cols, dtype=torch.bfloat16, device=device)
    step = max(1, (1 << 24) // max(cols, 1))          # bound int64 temporaries
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        idx = torch.arange(r0 * cols, r1 * cols, dtype=torch.int64, device=device)
        u = lowbias32((lowbias32(idx ^ k1) + k2) & _MASK32)
        t = tab[u >> (32 - TABLE_BITS)].view(r1 - r0, cols)
        out[r0:r1] = (t * gains[r0:r1, None]).to(torch.bfloat16)
    if outliers:
        ko = _key(seed, layer, matrix, "outliers")
        pos = lowbias32(torch.arange(outliers, dtype=torch.int64) ^ ko).numpy() % (rows * cols)
        sign = np.where(np.arange(outliers) % 2 == 0, 1.0, -1.0)
        for p_, s_ in zip(pos.tolist(), sign.tolist()):
            out.view(-1)[p_] = torch.tensor(s_ * 100.0 * SIGMA, dtype=torch.bfloat16)
    return out


def weights_rows(row_ids, rows: int, cols: int, seed: int = 0, layer: int = 0, matrix: int = 0,
                 dist: str = "t4", device="cpu") -> torch.Tensor:
    """The listed rows of ``weights(rows, cols, ...)`` (same bits; no planted outliers)."""
    device = torch.device(device)
    k1, k2 = _key(seed, layer, matrix, dist, "a"), _key(seed, layer, matrix, dist, "b")
    tab = _table(dist, device)
    gains = torch.from_numpy(row_gains(rows, seed, layer, matrix)).to(device)
    rid = torch.as_tensor(list(row_ids), dtype=torch.int64, device=device)
    idx = (rid[:, None] * cols + torch.arange(cols, dtype=torch.int64, device=device)[None, :]).reshape(-1)
    u = lowbias32((lowbias32(idx ^ k1) + k2) & _MASK32)
    t = tab[u >> (32 - TABLE_BITS)].view(rid.numel(), cols)
    return (t * gains[rid][:, None]).to(torch.bfloat16)


def block_weights(model: str, layer: int, seed: int = 0, dist: str = "t4", device="cpu",
                  outliers: bool = False):
    """The 7 bf16 matrices of decoder block ``layer`` of a Llama-shaped model."""
    out = []
    for m, (r, c) in enumerate(block_shapes(model)):
        n_out = 4 if (outliers and m == 6 and layer < 2) else 0
        out.append(weights(r, c, seed, layer, m, dist, device, outliers=n_out))
    return out


def random_codes_stream(n: int, seed: int, kind: str = "skewed") -> np.ndarray:
    """Byte symbol streams for codec fuzzing (uniform / skewed / uniform-subset)."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.integers(0, 256, n, dtype=np.uint8)
    if kind.startswith("subset"):
        k = int(kind[6:])
        alphabet = rng.permutation(256)[:k].astype(np.uint8)
        return alphabet[rng.integers(0, k, n)]
    if kind == "single":
        return np.full(n, rng.integers(0, 256), dtype=np.uint8)
    # skewed: geometric-like over a random permutation
    a = rng.permutation(256).astype(np.uint8)
    g = np.minimum(rng.geometric(rng.uniform(0.05, 0.9), n) - 1, 255)
    return a[g]
