"""Debug: R18 bf16 decode of the escape-heavy uniform stream — where does it differ?"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np, torch
import eqsynth, oracle as o, paper_2601_22787_b200 as eq
from test_gpu_parity import oracle_block_to_gpu, u16
for kind in ["uniform", "subset40", "skewed"]:
    s = eqsynth.random_codes_stream(64 * 4096, 3, kind)
    s = np.where((s & 0x7F) == 0x7F, s ^ 1, s).astype(np.uint8)
    S = (np.arange(64, dtype=np.uint16) * 37 + 0x3C00).astype(np.uint16)
    for pc in (o.CODEC_PAIR, o.CODEC_PAIR_G):
        blk = o.encode_codes([s.reshape(64, 4096)], [(64, 4096)], [S], 4096, codec=pc)
        print(kind, pc, "K", blk.pair.K, "fesc", blk.pair.fesc, "max pf", blk.pair.pf.max())
        v8 = eq.decode_dequant([oracle_block_to_gpu(blk)], eq.EQ_OUT_FP8)[0][0].view(torch.uint8).cpu().numpy().reshape(-1)
        print("  fp8 ok", (v8 == s).all())
        v = u16(eq.decode_dequant([oracle_block_to_gpu(blk)], eq.EQ_OUT_BF16)[0][0]).reshape(-1)
        ref = o.dequant(s.reshape(64, 4096), S).reshape(-1)
        bad = np.nonzero(v != ref)[0]
        print("  bf16 mismatches", bad.size)
        for i in bad[:12]:
            print("   ", i, "row", i // 4096, "col", i % 4096, "code", hex(s[i]), "got", hex(v[i]), "want", hex(ref[i]), "scale", hex(S[i // 4096]))
