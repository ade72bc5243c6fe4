"""ORACLE (test infrastructure only) for §8(f) NEXT row 3: the paper's scale optimisation
— "optimize each layer separately using L-BFGS ... we tune only the scale parameters S ...
We use the straight-through estimator for Q_γ", learning rate 0.25 for λ > 30 and
1.0 for λ ≤ 30, initialised with AbsMax (Alg. 1 l.1-2).

Plain numpy in fp64, following the algorithm step by step (reading R13):

* variables u_i = log2 s_i (one per output channel, positivity by construction, SPEC
  S:280); the scale actually used is s_i = RNE_bf16(2^u_i) (scales are stored in bf16 and
  the quantiser uses the stored value, R7);
* objective F(u) = Eq. 4 of the layer at those scales (R4): ΣD/‖W‖₁ + λ·ΣR/(M·N);
* gradient: the straight-through derivative (eqo_rd_row_fmt):
  ∂F/∂u_i = ln2 · s_i · ∂F/∂s_i,  ∂F/∂s_i = (A_i + B_i)/‖W‖₁ − λ·Q_i/(s_i·M·N);
* L-BFGS (Liu & Nocedal 1989, cited at P:191) with the two-loop recursion, history 10,
  H0 = γI with γ = sᵀy/yᵀy of the newest pair, pairs kept only if sᵀy > 1e-10 (torch);
  step: Armijo backtracking on the TRUE discrete objective, α_t = α0·2^-t, c1 = 1e-4,
  ≤ 32 backtracks; α0 = lr/‖d‖∞ for a steepest-descent direction (no curvature
  pairs yet: the largest log2-scale moves by lr) and α0 = lr for a quasi-Newton direction.
  (torch's first step lr·min(1, 1/‖g‖₁) is below the bf16 resolution of the scales in
  log space — F is piecewise constant in u — so no Armijo step would ever be accepted.)
  A non-descent direction resets the history to steepest descent;
* stops: ‖g‖∞ ≤ grad_tol or |ΔF| < change_tol or max|Δu| ≤ change_tol (converged), line
  search failure (not converged), or max_iters.

Pins: tests/test_oracle_lbfgs.py (two-loop = exact inverse-Hessian product on a quadratic
with a conjugate history; Rosenbrock; STE gradient = finite difference of the linearised
surrogate; on-grid fixed point; monotone trace; λ→∞ sparsity; Fig. A.1 monotonicity;
never below the exhaustive per-row optimum).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import FMT_E4M3, _u16, absmax_scales, l1 as _l1, lib, rd_row

LN2 = math.log(2.0)


def bf16_of_exp2(u: np.ndarray) -> np.ndarray:
    """s_i = RNE_bf16(2^u_i) (bit patterns)."""
    return np.array([lib().eqo_bf16_from_double(float(2.0 ** float(x))) for x in u], dtype=np.uint16)


def rd_eval(W, S, lam: float, fmt: int = FMT_E4M3, l1w: float | None = None):
    """Eq. 4 of one layer at bf16 scales S and its STE gradient w.r.t. u = log2 s.
    Returns (F, g[M], sums[M,5])."""
    W, S = _u16(W), _u16(S)
    M, N = W.shape
    if l1w is None:
        l1w = _l1(W)
    sums = np.stack([rd_row(W[i], int(S[i]), fmt) for i in range(M)])
    mn = float(M) * float(N)
    D, R, A, B, Q = (sums[:, k] for k in range(5))
    F = (D.sum() / l1w if l1w > 0 else 0.0) + lam * R.sum() / mn
    s = np.array([lib().eqo_bf16_to_double(int(x)) for x in S])
    g = LN2 * ((s * (A + B) / l1w if l1w > 0 else 0.0 * s) - lam * Q / mn)
    return F, g, sums


def two_loop(g: np.ndarray, hist: list) -> np.ndarray:
    """L-BFGS direction d = −H·g by the two-loop recursion; hist = [(s, y, rho)] oldest
    first, H0 = γI with γ = sᵀy/yᵀy of the newest pair."""
    q = -g.copy()
    al = []
    for s, y, rho in reversed(hist):
        a = rho * float(s @ q)
        q = q - a * y
        al.append(a)
    s_n, y_n, _ = hist[-1]
    r = q * (float(s_n @ y_n) / float(y_n @ y_n))
    for (s, y, rho), a in zip(hist, reversed(al)):
        b = rho * float(y @ r)
        r = r + s * (a - b)
    return r


@dataclass
class LbfgsResult:
    x: np.ndarray
    f: float
    trace: list = field(default_factory=list)     # F after every accepted step (F0 first)
    iterations: int = 0
    converged: bool = False
    evals: int = 0


def lbfgs_minimize(fun, x0: np.ndarray, max_iters: int = 100, history: int = 10, lr: float = 1.0,
                   c1: float = 1e-4, max_backtracks: int = 32, grad_tol: float = 1e-7,
                   change_tol: float = 1e-9) -> LbfgsResult:
    """Generic L-BFGS with Armijo backtracking; fun(x) -> (f, g)."""
    x = np.array(x0, dtype=np.float64)
    F, g = fun(x)
    res = LbfgsResult(x=x, f=F, trace=[F], evals=1)
    hist: list = []
    for k in range(max_iters):
        if np.max(np.abs(g)) <= grad_tol:
            res.converged = True
            break
        d = two_loop(g, hist) if hist else -g
        gd = float(g @ d)
        if gd >= 0.0:                                  # not a descent direction
            hist = []
            d = -g
            gd = float(g @ d)
        # steepest-descent steps (no curvature pairs yet) move the largest coordinate by lr;
        # quasi-Newton steps start at lr (R13)
        a0 = lr / float(np.max(np.abs(d))) if not hist else lr
        accepted = False
        for t in range(max_backtracks):
            a = a0 * 2.0 ** (-t)
            xn = x + a * d
            Fn, gn = fun(xn)
            res.evals += 1
            if Fn <= F + c1 * a * gd:
                accepted = True
                break
        if not accepted:
            res.converged = False
            break
        sk, yk = xn - x, gn - g
        ys = float(sk @ yk)
        if ys > 1e-10:
            hist.append((sk, yk, 1.0 / ys))
            if len(hist) > history:
                hist.pop(0)
        dF = F - Fn
        x, F, g = xn, Fn, gn
        res.trace.append(F)
        res.iterations = k + 1
        if abs(dF) < change_tol or float(np.max(np.abs(sk))) <= change_tol:
            res.converged = True
            break
    res.x, res.f = x, F
    return res


def default_lr(lam: float) -> float:
    """0.25 when λ > 30, 1.0 when λ ≤ 30 (applied to the R4-normalised λ)."""
    return 0.25 if lam > 30 else 1.0


def lbfgs_scales(W, lam: float, fmt: int = FMT_E4M3, max_iters: int = 100, history: int = 10,
                 lr: float | None = None, c1: float = 1e-4, max_backtracks: int = 32,
                 grad_tol: float = 1e-7, change_tol: float = 1e-9):
    """Alg. 1 l.2 by L-BFGS + STE for one layer: (S bf16 bits, LbfgsResult)."""
    W = _u16(W)
    l1w = _l1(W)
    s0 = absmax_scales(W, fmt=fmt)
    u0 = np.log2(np.array([lib().eqo_bf16_to_double(int(x)) for x in s0]))

    def fun(u):
        F, g, _ = rd_eval(W, bf16_of_exp2(u), lam, fmt, l1w)
        return F, g

    res = lbfgs_minimize(fun, u0, max_iters=max_iters, history=history,
                         lr=default_lr(lam) if lr is None else lr, c1=c1, max_backtracks=max_backtracks,
                         grad_tol=grad_tol, change_tol=change_tol)
    return bf16_of_exp2(res.x), res
