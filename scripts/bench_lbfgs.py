"""§8(f) NEXT row 3 measurements on one B200: L-BFGS + STE (eq_lbfgs_scales) vs the
exhaustive search (eq_search_scales) on one Llama-3-8B block — time, objective, effective
bits — and the λ <-> entropy curve of Fig. A.1 on synthetic weights."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import eqsynth  # noqa: E402
import paper_2601_22787_b200 as eq  # noqa: E402


def entropy_bits(Ws, scales):
    h = torch.zeros(256, dtype=torch.int64, device=Ws[0].device)
    r0 = 0
    for W in Ws:
        eq.quantize_hist(W, scales[r0:r0 + W.shape[0]], codes=False, hist=h)
        r0 += W.shape[0]
    p = h.double() / h.sum()
    p = p[p > 0]
    return float(-(p * p.log2()).sum())


def main():
    dev = torch.device("cuda")
    Ws = eqsynth.block_weights("llama-3-8b", 0, device=dev)
    out = {"workload": "one Llama-3-8B block (7 layers, 218 M weights), synthetic t4 weights"}
    for lam in (30.0, 230.2):
        torch.cuda.synchronize()
        t0 = time.time()
        sc, tr, info = eq.lbfgs_scales(Ws, lam)
        torch.cuda.synchronize()
        t_l = time.time() - t0
        t0 = time.time()
        se = torch.cat([eq.search_scales(W, [lam])[0] for W in Ws])
        torch.cuda.synchronize()
        t_e = time.time() - t0
        trn = tr.cpu().numpy()
        fl = [float(t[~np.isnan(t)][-1]) for t in trn]
        f0 = [float(t[0]) for t in trn]
        fe = [float(eq.search_scales(W, [lam], with_obj=True)[1][0].sum()) for W in Ws]
        out[f"lambda_{lam}"] = {
            "lbfgs_s": t_l, "exhaustive_s": t_e, "lbfgs_iters": info[:, 0].tolist(),
            "lbfgs_passes": info[:, 2].tolist(), "converged": info[:, 1].tolist(),
            "objective_absmax": f0, "objective_lbfgs": fl, "objective_exhaustive": fe,
            "entropy_lbfgs": entropy_bits(Ws, sc), "entropy_exhaustive": entropy_bits(Ws, se)}
    # Fig. A.1: λ vs entropy (q_proj + gate_proj of block 0, L-BFGS), log-spaced λ
    sweep = []
    for lam in (1.0, 3.0, 10.0, 30.0, 100.0, 300.0, 1000.0):
        sel = [Ws[0], Ws[4]]
        sc, _, _ = eq.lbfgs_scales(sel, lam)
        se = torch.cat([eq.search_scales(W, [lam])[0] for W in sel])
        sweep.append({"lambda": lam, "entropy_lbfgs": entropy_bits(sel, sc), "entropy_exhaustive": entropy_bits(sel, se)})
    out["fig_a1_sweep"] = sweep
    print(json.dumps(out))


if __name__ == "__main__":
    main()
