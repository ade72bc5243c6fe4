"""Single-block decode latency vs chunk length (the paper's one-block-at-a-time inference,
P:521): one Llama-3-8B-shaped block, word codec, bf16 out, CUDA-event timed."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import eqsynth  # noqa: E402
import paper_2601_22787_b200 as eq  # noqa: E402


def main():
    dev = torch.device("cuda")
    Ws = eqsynth.block_weights("llama-3-8b", 0, device=dev)
    out = {"workload": "one llama-3-8b-shaped block (218 M weights), word codec, lambda 230.2, bf16 out"}
    for cs in (4096, 2048, 1024, 512):
        blk = eq.quantize_encode(Ws, lam=230.2, chunk_symbols=cs, codec=eq.EQ_CODEC_WORD)
        dec = eq.Decoder([blk], eq.EQ_OUT_BF16)
        for _ in range(3):
            dec()
        dec.check()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            dec()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 20
        out[f"cs{cs}"] = {"ms": ms, "chunks": blk.n_chunks, "effective_bits": blk.effective_bits(),
                          "gbs": (blk.compressed_bytes() + 2 * blk.n_params) / (ms / 1e3) / 1e9}
        del dec, blk
    print(json.dumps(out))


if __name__ == "__main__":
    main()
