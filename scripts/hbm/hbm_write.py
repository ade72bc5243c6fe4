"""Write-dominated HBM bandwidth on this B200 (context for the decoder's roofline): the
decoder writes 13.96 GB and reads 2.2 GB per launch, so its ceiling is the write path, not the
read+write copy bandwidth of MEASURED_PEAKS.json.  Builds scripts/hbm/hbm_write.cu with nvcc."""
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
for f in ("hbm_write256", "hbm_write128"):
    getattr(L, f).argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
L.hbm_mix18.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]


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


nbytes = 14_000_000_000 // 256 * 256
dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
src = torch.empty(nbytes // 8, dtype=torch.uint8, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream
out = {"bytes_written": nbytes}
for blocks_per_sm in (4, 8, 16):
    g = sms * blocks_per_sm
    ms = timed(lambda: L.hbm_write256(dst.data_ptr(), nbytes, g, 256, st))
    out[f"write256_{blocks_per_sm}x256_GBs"] = nbytes / ms / 1e6
    ms = timed(lambda: L.hbm_write128(dst.data_ptr(), nbytes, g, 256, st))
    out[f"write128_{blocks_per_sm}x256_GBs"] = nbytes / ms / 1e6
    ms = timed(lambda: L.hbm_mix18(src.data_ptr(), dst.data_ptr(), nbytes, g, 256, st))
    out[f"mix1to8_{blocks_per_sm}x256_GBs"] = (nbytes + nbytes / 8) / ms / 1e6
ms = timed(lambda: dst.fill_(1))
out["torch_fill_GBs"] = nbytes / ms / 1e6
ms = timed(lambda: dst[: nbytes // 2].copy_(dst[nbytes // 2:]))
out["torch_copy_read_write_GBs"] = nbytes / ms / 1e6
print(json.dumps(out))
