"""Builds libentquant.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun)."""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libentquant.so")
SOURCES = ["rans_dec.cu", "quant.cu", "table.cu", "rans_enc.cu", "api.cu", "qmatmul.cu", "lbfgs.cu", "crc.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-ftz=false", "-prec-div=true",
              "-prec-sqrt=true", "-fmad=false"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "entquant.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines=(), so: str | None = None) -> str:
    """Compile and link.  ``defines``/``so`` produce alternative builds for A/B experiments."""
    target = so or SO
    if not force and not defines and not stale():
        return SO
    objs = []
    tmp = tempfile.mkdtemp(prefix="eqbuild_")       # per-build object dir: parallel variant builds never collide
    for s in SOURCES:
        o = os.path.join(tmp, s.replace(".cu", ".o"))
        cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        objs.append(o)
    subprocess.check_call([_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", target + ".tmp",
                           *objs, "-cudart", "static"])
    os.replace(target + ".tmp", target)
    for o in objs:
        os.remove(o)
    os.rmdir(tmp)
    return target


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[len("--so="):] for a in sys.argv[1:] if a.startswith("--so=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, so=outs[0] if outs else None))
