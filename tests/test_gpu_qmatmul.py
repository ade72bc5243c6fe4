"""NEXT row 1 / config 4: decode fused into a tcgen05 GEMM.  y = x · Ŵᵀ where Ŵ is the
oracle's exact dequantised weight matrix; fp32 tensor-core accumulation differs from the
fp64 reference only by rounding (bound: 1e-4 · Σ_k |x_k ŵ_k| per output)."""
import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
import paper_2601_22787_b200 as eq

pytestmark = pytest.mark.gpu
DEV = "cuda"


def to_gpu_block(blk):
    from test_gpu_parity import oracle_block_to_gpu
    return oracle_block_to_gpu(blk)            # incl. the pair codec's 512-entry table buffer


@pytest.mark.parametrize("codec", [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G])
@pytest.mark.parametrize("cs,fmt", [(4096, 0), (2048, 0), (1024, 1), (256, 0)])
@pytest.mark.parametrize("batch", [1, 8, 61])
def test_qmatmul_matches_fp64_reference(cs, fmt, batch, codec):
    shapes = [(256, 4096), (128, 2048 if cs <= 2048 else 4096)]
    Ws = [eqsynth.weights(r, c, seed=31, layer=0, matrix=m) for m, (r, c) in enumerate(shapes)]
    S = [(o.absmax_scales(W, fmt).astype(np.int32) + 128 * 12).astype(np.uint16) for W in Ws]
    blk = o.quantize_encode(Ws, scales=S, cs=cs, fmt=fmt, codec=codec)
    g = to_gpu_block(blk)
    What = [d.view(np.int16) for d in o.decode_dequant(blk)]
    for layer, (r, c) in enumerate(shapes):
        x = (torch.randn(batch, c, generator=torch.Generator().manual_seed(layer + batch)) * 0.5).to(torch.bfloat16)
        W64 = torch.from_numpy(What[layer]).view(torch.bfloat16).double().numpy()
        X64 = x.double().numpy()
        ref = X64 @ W64.T
        bound = 1e-4 * (np.abs(X64) @ np.abs(W64).T) + 1e-30
        for rep in range(3):              # repeated launches: catches staging races
            y = eq.qmatmul(g, layer, x.to(DEV)).cpu().double().numpy()
            assert (np.abs(y - ref) <= bound).all(), (layer, rep, float(np.max(np.abs(y - ref) / bound)))


@pytest.mark.parametrize("codec", [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G])
def test_qmatmul_shape_errors_and_corruption(codec):
    Ws = [eqsynth.weights(128, 4096, seed=3)]
    blk = o.quantize_encode(Ws, scales=[o.absmax_scales(Ws[0])], cs=4096, codec=codec)
    g = to_gpu_block(blk)
    with pytest.raises(eq.EqError):
        eq.qmatmul(g, 0, torch.zeros(2, 4000, dtype=torch.bfloat16, device=DEV))
    blk2 = o.quantize_encode([eqsynth.weights(128, 4096, seed=4)], lam=None, cs=3000)
    with pytest.raises(eq.EqError) as ei:
        eq.qmatmul(to_gpu_block(blk2), 0, torch.zeros(2, 4096, dtype=torch.bfloat16, device=DEV))
    assert ei.value.status == eq.EQ_ERR_SHAPE
    g.payload[100] ^= 0x77
    with pytest.raises(eq.EqError) as ei:
        eq.qmatmul(g, 0, torch.ones(2, 4096, dtype=torch.bfloat16, device=DEV))
    assert ei.value.status == eq.EQ_ERR_CORRUPT


@pytest.mark.parametrize("codec", [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G])
@pytest.mark.parametrize("batch", [1, 24])
def test_qmatmul_group_one_launch_deterministic(batch, codec):
    """All layers of a block in one grouped launch (mixed chunk counts per row: split-K
    partials for some, direct output for others), bitwise repeatable, each vs fp64."""
    shapes = [(256, 1024), (128, 2048), (384, 1024), (128, 3072)]
    Ws = [eqsynth.weights(r, c, seed=77, layer=1, matrix=m) for m, (r, c) in enumerate(shapes)]
    blk = o.quantize_encode(Ws, lam=None, cs=1024, codec=codec)
    g = to_gpu_block(blk)
    What = o.decode_dequant(blk)
    xs = [(torch.randn(batch, c, generator=torch.Generator().manual_seed(5 + m)) * 0.3).to(torch.bfloat16)
          for m, (_, c) in enumerate(shapes)]
    order = [3, 0, 2, 1]                       # any order of layers
    ys = eq.qmatmul_group(g, order, [xs[l].to(DEV) for l in order])
    again = eq.qmatmul_group(g, order, [xs[l].to(DEV) for l in order])
    for l, y, y2 in zip(order, ys, again):
        assert torch.equal(y, y2)
        W64 = torch.from_numpy(What[l]).view(torch.bfloat16).double().numpy()
        X64 = xs[l].double().numpy()
        ref = X64 @ W64.T
        bound = 1e-4 * (np.abs(X64) @ np.abs(W64).T) + 1e-30
        assert (np.abs(y.cpu().double().numpy() - ref) <= bound).all(), l


def test_qmatmul_workspace_contract():
    shapes = [(128, 2048)]
    Ws = [eqsynth.weights(128, 2048, seed=9)]
    g = to_gpu_block(o.quantize_encode(Ws, lam=None, cs=512))
    x = torch.ones(3, 2048, dtype=torch.bfloat16, device=DEV)
    small = torch.empty(16, dtype=torch.uint8, device=DEV)
    b = g.c_struct()
    import ctypes
    la = (ctypes.c_uint32 * 1)(0)
    need = eq.lib().eq_qmatmul_workspace_bytes(ctypes.byref(b), 1, la, 3)
    assert need >= 4 * 3 * 128 * 4
    y = torch.empty(3, 128, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    xa = (ctypes.c_void_p * 1)(x.data_ptr())
    ya = (ctypes.c_void_p * 1)(y.data_ptr())
    st = eq.lib().eq_qmatmul_group(ctypes.byref(b), 1, la, xa, ya, 3, small.data_ptr(), 16, err.data_ptr(), None)
    assert st == eq.EQ_ERR_BUFFER


@pytest.mark.parametrize("codec", [o.CODEC_BYTE, o.CODEC_WORD, o.CODEC_PAIR, o.CODEC_PAIR_G])
def test_qmatmul_runaway_stream_is_reported_not_overread(codec):
    """A chunk whose state is forced to 1 consumes a renormalisation unit at every symbol and
    runs far past its end: the fused kernel must stop reading it (no access beyond the
    payload slack) and report EQ_ERR_CORRUPT; the other chunks still decode."""
    Ws = [eqsynth.weights(128, 4096, seed=12)]
    blk = o.quantize_encode(Ws, scales=[(o.absmax_scales(Ws[0]).astype(np.int32) + 1700).astype(np.uint16)],
                            cs=2048, codec=codec)
    g = to_gpu_block(blk)
    last = blk.n_chunks - 1                                  # the chunk next to the payload end
    a = int(blk.chunk_off[last])
    g.payload[a:a + 4] = torch.tensor([1, 0, 0, 0], dtype=torch.uint8, device=DEV)
    with pytest.raises(eq.EqError) as ei:
        eq.qmatmul(g, 0, torch.ones(4, 4096, dtype=torch.bfloat16, device=DEV))
    assert ei.value.status == eq.EQ_ERR_CORRUPT
    d = eq.Decoder([g], eq.EQ_OUT_BF16)
    d()
    with pytest.raises(eq.EqError) as ei:
        d.check()
    assert ei.value.status == eq.EQ_ERR_CORRUPT
