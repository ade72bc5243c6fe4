"""Block-pipelined inference measurement (NEXT row 2): time of a Llama-3-8B-shaped linear
forward over the 32 blocks with (a) resident bf16 weights, (b) the paper's single decode
buffer (decode then forward), (c) S-slot pipelining (decode of upcoming blocks on a
side stream).  One JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import eqsynth  # noqa: E402
import paper_2601_22787_b200 as eq  # noqa: E402
from paper_2601_22787_b200.pipeline import BlockPipeline, llama_block_forward, llama_block_forward_fused  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("model", nargs="?", default="llama-3-8b")
    ap.add_argument("--codec", default="pair", choices=["word", "pair", "pairg"])
    ap.add_argument("--cs", type=int, default=4096)
    args = ap.parse_args()
    model = args.model
    nb = eqsynth.LLAMA[model]["layers"]
    dev = torch.device("cuda")
    lam = 230.2
    codec = {"word": eq.EQ_CODEC_WORD, "pair": eq.EQ_CODEC_PAIR, "pairg": eq.EQ_CODEC_PAIR_G}[args.codec]
    blocks, dense = [], []
    for lid in range(nb):
        Ws = eqsynth.block_weights(model, lid, device=dev)
        blocks.append(eq.quantize_encode(Ws, lam=lam, codec=codec, chunk_symbols=args.cs, chunk_mode=eq.EQ_CHUNK_ROW))
        dense.append(Ws)
    hid = eqsynth.LLAMA[model]["hidden"]
    out = {"workload": f"{model}-shaped linear forward over {nb} blocks (decode-in-the-loop, bf16 weights, "
                       f"{args.codec} codec, row chunks of {args.cs})",
           "effective_bits": sum(b.compressed_bytes() for b in blocks) * 8 / sum(b.n_params for b in blocks)}
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(1 << 26, dtype=torch.uint8, device=dev)
    for batch in (1, 64):
        x0 = torch.randn(batch, hid, device=dev, dtype=torch.bfloat16) * 0.1

        def f_dense():
            x = x0
            for Ws in dense:
                x = llama_block_forward(Ws, x)
            return x
        r = {"dense_bf16_ms": timed(f_dense)}

        def f_fused():                          # every GEMM fused with its decode, 4 launches per block
            x = x0
            for b in blocks:
                x = llama_block_forward_fused(b, x, err, ws)
            return x
        r["fused_gemm_ms"] = timed(f_fused)
        assert int(err.item()) == 0
        for group, slots in ((1, 1), (1, 2), (4, 1), (4, 2), (8, 2), (16, 2), (nb, 1)):
            pipe = BlockPipeline(blocks, slots=slots, group=group)
            r[f"decode_g{group}_s{slots}_ms"] = timed(lambda: pipe.run(lambda k, v, x: llama_block_forward(v, x), x0))
            pipe.check()
            del pipe
            torch.cuda.empty_cache()
        out[f"batch{batch}"] = r
    dec1 = eq.Decoder([blocks[0]])
    out["single_block_decode_ms"] = timed(lambda: dec1())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
