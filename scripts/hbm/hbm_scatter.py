"""The decoder's write pattern without the decode: 1.7 M threads (chunks), each writing its own
8 KB region front to back in 32-byte (or 4 × 32-byte) steps, with / without evict-first."""
import ctypes
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libhbm_write.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       os.path.join(HERE, "hbm_write.cu"), "-o", SO])
L = ctypes.CDLL(SO)
L.hbm_scatter.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                          ctypes.c_void_p]


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


region = 8192
threads = 1703936                                   # the 8B set's chunks at 4096 symbols (bf16: 8 KB each)
dst = torch.empty(region * threads, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
out = {"bytes": region * threads}
for burst in (1, 4):
    for ef in (1, 0):
        ms = timed(lambda: L.hbm_scatter(dst.data_ptr(), region, threads, burst, ef, 256, st))
        out[f"scatter_burst{burst}_ef{ef}_GBs"] = region * threads / ms / 1e6
print(json.dumps(out))
