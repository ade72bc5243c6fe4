"""§8(f) NEXT row 3 on the GPU: L-BFGS + STE scale optimisation (eq_lbfgs_scales,
eq_rd_eval) against the fp64 oracle (oracle/lbfgs.py).  Every term is the same exact or
correctly rounded f64 operation on both sides and only summation orders differ, so the
trajectories agree exactly: identical bf16 scales, iteration counts and stop reasons,
traces within 1e-12 relative."""
import math

import numpy as np
import pytest
import torch

import eqsynth
import oracle as o
from oracle import lbfgs as L
import paper_2601_22787_b200 as eq

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _bf16_bits(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("mult", [1.0, 37.0, 0.3, 3000.0])
def test_rd_eval_matches_oracle(fmt, mult):
    W = eqsynth.weights(40, 333, seed=21)
    s0 = o.absmax_scales(W, fmt=fmt)
    S = np.array([o.lib().eqo_bf16_from_double(o.lib().eqo_bf16_to_double(int(x)) * mult) for x in s0], dtype=np.uint16)
    lam = 77.0
    F, g, sums = L.rd_eval(W, S, lam, fmt)
    f_gpu, g_gpu = eq.rd_eval(W.to(DEV), torch.from_numpy(S.view(np.int16)).view(torch.bfloat16).to(DEV), lam, format=fmt)
    assert f_gpu.item() == pytest.approx(F, rel=1e-12)
    l1w = o.l1(W)
    s = np.array([o.lib().eqo_bf16_to_double(int(x)) for x in S])
    scale = math.log(2.0) * (np.abs(s * (sums[:, 2] + sums[:, 3]) / l1w) + lam * sums[:, 4] / (W.numel()))
    assert np.all(np.abs(g_gpu.cpu().numpy() - g) <= 1e-12 * scale + 1e-300)


CASES = [
    ([(64, 256), (128, 96), (32, 512)], 230.2, 0),
    ([(48, 200), (16, 1024)], 12.0, 0),
    ([(64, 128)], 0.0, 0),
    ([(96, 160), (40, 64)], 40.0, 1),
]


@pytest.mark.parametrize("shapes,lam,fmt", CASES)
def test_lbfgs_trajectory_matches_oracle(shapes, lam, fmt):
    Ws = [eqsynth.weights(r, c, seed=3, layer=1, matrix=m) for m, (r, c) in enumerate(shapes)]
    scales, trace, info = eq.lbfgs_scales([W.to(DEV) for W in Ws], lam, format=fmt, max_iters=60)
    sg = _bf16_bits(scales)
    tr = trace.cpu().numpy()
    inf = info.cpu().numpy()
    r0 = 0
    for i, W in enumerate(Ws):
        S, res = L.lbfgs_scales(W, lam, fmt=fmt, max_iters=60)
        M = W.shape[0]
        assert np.array_equal(sg[r0:r0 + M], S), (i, int((sg[r0:r0 + M] != S).sum()))
        assert inf[i, 0] == res.iterations and bool(inf[i, 1]) == res.converged, (i, inf[i], res.iterations)
        n = len(res.trace)
        assert np.allclose(tr[i, :n], res.trace, rtol=1e-12, atol=0), i
        assert np.all(np.isnan(tr[i, n:]))
        r0 += M


def test_lbfgs_config1_deterministic_and_above_exhaustive():
    W = eqsynth.weights(256, 256, seed=0)
    a = eq.lbfgs_scales([W.to(DEV)], 230.2)
    b = eq.lbfgs_scales([W.to(DEV)], 230.2)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1].nan_to_num(), b[1].nan_to_num())
    S, res = L.lbfgs_scales(W, 230.2)
    assert np.array_equal(_bf16_bits(a[0]), S)
    Se, _ = o.search(W, 230.2)
    f_l = o.objective(W, _bf16_bits(a[0]), 230.2)
    assert f_l >= o.objective(W, Se, 230.2) - 1e-12
    assert f_l < 1.1 * o.objective(W, Se, 230.2)


def test_lbfgs_llama_block_invariants():
    """Full Llama-3-8B block (7 layers, one call): monotone traces, large improvement over
    AbsMax, never below the GPU exhaustive search's per-row optimum."""
    Ws = eqsynth.block_weights("llama-3-8b", 0, device=DEV)
    lam = 230.2
    scales, trace, info = eq.lbfgs_scales(Ws, lam, max_iters=100)
    tr = trace.cpu().numpy()
    r0 = 0
    for i, W in enumerate(Ws):
        t = tr[i][~np.isnan(tr[i])]
        assert np.all(np.diff(t) <= 0)
        assert t[-1] < 0.01 * t[0]
        _, fe = eq.search_scales(W, [lam], with_obj=True)
        assert t[-1] >= float(fe[0].sum().item()) * (1 - 1e-9)
        r0 += W.shape[0]


def test_lbfgs_argument_errors():
    W = torch.zeros(8, 8, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(eq.EqError):
        eq.lbfgs_scales([W], -1.0)
    with pytest.raises(eq.EqError):
        eq.lbfgs_scales([W], 1.0, history=0)
    # an all-zero layer: AbsMax scales 1, gradient 0 -> converged at iteration 0
    s, tr, info = eq.lbfgs_scales([W], 5.0)
    assert torch.all(s == 1.0) and info[0, 0].item() == 0 and info[0, 1].item() == 1
