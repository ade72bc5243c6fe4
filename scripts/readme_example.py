"""The README's Python API example (run on a GPU box to check it)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, eqsynth, paper_2601_22787_b200 as eq
Ws = eqsynth.block_weights("llama-3-8b", 0, device="cuda")        # 7 bf16 matrices of one block
lam, _ = eq.calibrate_lambda(Ws, 2.0)                             # global λ for ~2 bits/param
blk = eq.quantize_encode(Ws, lam=lam, chunk_mode=eq.EQ_CHUNK_ROW)  # Alg. 1 (pair codec by default)
views = eq.decode_dequant([blk])[0]                               # Alg. 2: bf16 views into an arena
ys = eq.qmatmul_group(blk, list(range(7)),                        # decode fused into tcgen05 GEMMs
                      [torch.randn(1, W.shape[1], device="cuda", dtype=torch.bfloat16) for W in Ws])
torch.cuda.synchronize()
print("readme example ok:", len(views), [tuple(y.shape) for y in ys], "%.3f bits" % blk.effective_bits())
