"""Config 4: one Llama-3-8B decoder block (7 linears) — fused decode→tcgen05 GEMM
(eq_qmatmul_group) vs decode-then-cuBLAS, batch 1 and 64.  Default: the bench's pair codec with
ROW chunking at 4096 symbols (4096+4096+4096+2048 per down_proj row), i.e. the same encoding
as config 3; reports the fused launch's decode rate (symbols / s)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import eqsynth  # noqa: E402
import paper_2601_22787_b200 as eq  # noqa: E402


def timed(fn, reps=20, warm=3):
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
    ap.add_argument("--cs", type=int, default=4096)
    ap.add_argument("--chunk-mode", default="row", choices=["row", "layer"])
    ap.add_argument("--profile", action="store_true", help="one grouped launch per batch (for ncu)")
    ap.add_argument("--codec", default="pair", choices=["byte", "word", "pair", "pairg"])
    args = ap.parse_args()
    codec = {"byte": eq.EQ_CODEC_BYTE, "word": eq.EQ_CODEC_WORD, "pair": eq.EQ_CODEC_PAIR, "pairg": eq.EQ_CODEC_PAIR_G}[args.codec]
    mode = {"row": eq.EQ_CHUNK_ROW, "layer": eq.EQ_CHUNK_LAYER}[args.chunk_mode]
    dev = torch.device("cuda")
    Ws = eqsynth.block_weights("llama-3-8b", 0, device=dev)
    blk = eq.quantize_encode(Ws, lam=230.2, chunk_symbols=args.cs, codec=codec, chunk_mode=mode)
    dec = eq.Decoder([blk])
    out = {"workload": f"config4: Llama-3-8B decoder block (q,k,v,o,gate,up,down), chunk {args.cs} "
                       f"({args.chunk_mode} chunking), ~2 bits, {args.codec} codec",
           "effective_bits": blk.effective_bits(), "params": blk.n_params, "chunks": blk.n_chunks}
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    for batch in (1, 64):
        xs = [torch.randn(batch, c, device=dev, dtype=torch.bfloat16) * 0.1 for _, c in blk.shapes]
        ys = [torch.empty(batch, r, device=dev) for r, _ in blk.shapes]

        ws = torch.empty(1 << 26, dtype=torch.uint8, device=dev)
        ys_grp = [torch.empty(batch, r, device=dev) for r, _ in blk.shapes]

        def fused_group():                      # all 7 GEMMs of the block in one launch
            eq.qmatmul_group(blk, list(range(7)), xs, ys_grp, err=err, check=False, workspace=ws)

        def fused_chain():                      # Llama dataflow: {q,k,v} -> o -> {gate,up} -> down
            for ls in ([0, 1, 2], [3], [4, 5], [6]):
                eq.qmatmul_group(blk, ls, [xs[l] for l in ls], [ys[l] for l in ls], err=err, check=False,
                                 workspace=ws)

        if args.profile:
            fused_group()
            torch.cuda.synchronize()
            continue

        def fused():
            for l in range(7):
                eq.qmatmul(blk, l, xs[l], ys[l], err=err, check=False, workspace=ws)

        def unfused():
            dec()
            vs = dec.views()[0]
            for l in range(7):
                torch.matmul(xs[l], vs[l].t())

        def dense():
            for l in range(7):
                torch.matmul(xs[l], Ws[l].t())
        out[f"batch{batch}"] = {"fused_group_ms": timed(fused_group), "fused_chain4_ms": timed(fused_chain),
                                "fused_per_layer_ms": timed(fused), "decode_then_cublas_ms": timed(unfused),
                                "dense_bf16_cublas_ms": timed(dense)}
        out[f"batch{batch}"]["fused_group_decode_Tsym_per_s"] = blk.n_params / out[f"batch{batch}"]["fused_group_ms"] / 1e9
        out[f"batch{batch}"]["decode_only_ms"] = timed(dec)
        eq.check(err)
        # correctness vs decode + fp32 matmul
        dec()
        vs = dec.views()[0]
        for l in range(7):
            eq.qmatmul(blk, l, xs[l], ys[l])
            out[f"batch{batch}"][f"group_equals_single_layer{l}"] = bool(torch.equal(ys[l], ys_grp[l]))
            ref = xs[l].float() @ vs[l].float().t()
            rel = ((ys[l] - ref).abs().max() / ref.abs().max()).item()
            out[f"batch{batch}"][f"maxrel_layer{l}"] = rel
    print(json.dumps(out))


if __name__ == "__main__":
    main()
