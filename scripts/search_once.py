"""One exhaustive scale search (a2, Eq. 4) over a Llama-3-8B q_proj on cuda:0 — an ncu target."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import eqsynth  # noqa: E402
import paper_2601_22787_b200 as eq  # noqa: E402

dev = torch.device("cuda")
W = eqsynth.weights(4096, 4096, seed=0, layer=0, matrix=0, device=dev)
eq.quantize_encode([W], lam=230.2)
torch.cuda.synchronize()
t = time.time()
eq.quantize_encode([W], lam=230.2)
torch.cuda.synchronize()
print("encode 4096x4096: %.3f s" % (time.time() - t))
