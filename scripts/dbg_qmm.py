import sys, os
sys.path.insert(0, os.getcwd())
import torch, eqsynth, paper_2601_22787_b200 as eq
dev = torch.device("cuda")
Ws = eqsynth.block_weights("llama-3-8b", 0, device=dev)
blk = eq.quantize_encode(Ws, lam=230.2, chunk_symbols=2048)
dec = eq.Decoder([blk]); dec(); dec.check(); print("decode ok")
for batch in (1, 64):
    for l in range(7):
        x = torch.randn(batch, blk.shapes[l][1], device=dev, dtype=torch.bfloat16) * 0.1
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        y = eq.qmatmul(blk, l, x, err=err, check=False)
        torch.cuda.synchronize()
        e = int(err.item())
        ref = x.float() @ dec.views()[0][l].float().t()
        rel = ((y - ref).abs().max() / ref.abs().max()).item()
        print(batch, l, blk.shapes[l], "err", e, "rel", rel)
