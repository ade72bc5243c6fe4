"""HBM write-only bandwidth vs copy bandwidth on this B200 (context for the decoder's roofline:
its traffic is 86 % writes).  torch fill_ (write-only) and copy_ (read + write) of ~14 GB."""
import json
import torch


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


n = 14_000_000_000 // 2
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
src = torch.empty(n // 8, dtype=torch.bfloat16, device="cuda")
out = {}
ms = timed(lambda: a.fill_(1.0))
out["fill_write_only_GBs"] = 2 * n / ms / 1e6
ms = timed(lambda: b.copy_(a))
out["copy_read_write_GBs"] = 4 * n / ms / 1e6
# 1 : 8 read : write mix (the decoder's 1.75 GB in : 14 GB out): expand a small source 8x
ms = timed(lambda: a.view(8, n // 8).copy_(src.expand(8, n // 8)))
out["expand_1to8_GBs"] = (2 * n / 8 + 2 * n) / ms / 1e6
print(json.dumps(out))
