"""CPU-side checks of the boundary: the C-ABI library builds/loads and exports every
symbol include/entquant.h declares; host-only entry points (no device work) behave."""
import ctypes
import os
import re

import pytest

import paper_2601_22787_b200 as eq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "entquant.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_22787_b200 import build
    build.build()
    return eq.lib()


def test_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(eq.EXPORTS)


def test_status_strings_and_version(lib):
    assert eq.status_string(eq.EQ_ERR_CORRUPT) == "corrupt"
    assert eq.status_string(eq.EQ_ERR_UNREACHABLE_TARGET) == "unreachable-target"
    assert "sm_100a" in eq.version()


def test_encode_bounds_host_only(lib):
    t = (eq.eq_tensor * 2)(eq.eq_tensor(1, 4096, 4096), eq.eq_tensor(1, 14336, 4096))
    p = eq._params()
    cap, nc, sb = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint64()
    assert lib.eq_encode_bounds(t, 2, ctypes.byref(p), ctypes.byref(cap), ctypes.byref(nc), ctypes.byref(sb)) == 0
    assert nc.value == (4096 * 4096 + 14336 * 4096) // 4096
    assert cap.value >= 4 * nc.value + 2 * (4096 * 4096 + 14336 * 4096) + 16
    assert sb.value >= 4096 * 4096 + 14336 * 4096
    bad = (eq.eq_tensor * 1)(eq.eq_tensor(1, 0, 5))
    assert lib.eq_encode_bounds(bad, 1, ctypes.byref(p), None, None, None) == eq.EQ_ERR_SHAPE
    p.prob_bits = 11
    assert lib.eq_encode_bounds(t, 2, ctypes.byref(p), None, None, None) == eq.EQ_ERR_ARG


def test_arena_layout_host_only(lib):
    b = eq.eq_block()
    b.n_layers = 3
    for i, (r, c) in enumerate([(37, 53), (1, 1), (64, 64)]):
        b.layer_rows[i], b.layer_cols[i] = r, c
    offs = (ctypes.c_uint64 * 8)()
    tot = ctypes.c_uint64()
    assert lib.eq_arena_layout(ctypes.byref(b), 1, eq.EQ_OUT_BF16, offs, ctypes.byref(tot)) == 0
    assert list(offs[:3]) == [0, 4096, 4352]
    assert tot.value == 4352 + 64 * 64 * 2
    assert all(o % eq.EQ_ARENA_ALIGN == 0 for o in offs[:3])
    assert lib.eq_arena_layout(ctypes.byref(b), 1, 7, offs, ctypes.byref(tot)) == eq.EQ_ERR_ARG


def test_compute_calls_need_cuda_tensors():
    import torch
    with pytest.raises((RuntimeError, ValueError)):
        eq.absmax(torch.zeros(4, 4, dtype=torch.bfloat16))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2601_22787_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                for pat in ("import oracle", "from oracle", "liboracle", "eq_oracle", "eqo_"):
                    assert pat not in src, (f, pat)


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of eq_params / eq_block / eq_lbfgs_params have the C layout
    (sizes and every field offset, from a gcc-compiled probe of include/entquant.h)."""
    import subprocess
    structs = {"eq_params": eq.eq_params, "eq_block": eq.eq_block, "eq_lbfgs_params": eq.eq_lbfgs_params,
               "eq_tensor": eq.eq_tensor}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "entquant.h"', 'int main(void) {']
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            cf = "lambda" if f == "lambda_" else f
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {cf}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, f"{name}.{f}"


def test_codec_parameter_validated(lib):
    t = (eq.eq_tensor * 1)(eq.eq_tensor(1, 64, 64))
    p = eq._params(codec=eq.EQ_CODEC_WORD)
    assert lib.eq_encode_bounds(t, 1, ctypes.byref(p), None, None, None) == 0
    p.codec = eq.EQ_CODEC_PAIR
    assert lib.eq_encode_bounds(t, 1, ctypes.byref(p), None, None, None) == 0
    p.codec = eq.EQ_CODEC_PAIR_G
    assert lib.eq_encode_bounds(t, 1, ctypes.byref(p), None, None, None) == 0
    p.codec = 4
    assert lib.eq_encode_bounds(t, 1, ctypes.byref(p), None, None, None) == eq.EQ_ERR_ARG


def test_crc32_host_side(lib):
    """eq_crc32's host-side contract without a GPU: scratch size (4 bytes per 4 KB piece + 16),
    argument errors before any launch."""
    assert lib.eq_crc32_scratch_bytes(0) == 16
    assert lib.eq_crc32_scratch_bytes(1) == 20
    assert lib.eq_crc32_scratch_bytes(4096) == 20
    assert lib.eq_crc32_scratch_bytes(4097) == 24
    assert lib.eq_crc32(None, 10, None, None, 0, None) == eq.EQ_ERR_ARG
    assert lib.eq_crc32(None, 10, ctypes.c_void_p(16), None, 0, None) == eq.EQ_ERR_ARG
    assert lib.eq_crc32(ctypes.c_void_p(16), 8192, ctypes.c_void_p(16), ctypes.c_void_p(16), 8, None) == eq.EQ_ERR_BUFFER


def test_header_constants_match_the_binding():
    """Every #define EQ_* integer constant of include/entquant.h that the binding also names has
    the binding's value (the codecs, chunk modes, formats, output types, status codes...)."""
    import re
    hdr = open(os.path.join(ROOT, "include", "entquant.h")).read()
    defs = {m.group(1): int(m.group(2), 0) for m in re.finditer(r"#define\s+(EQ_[A-Z0-9_]+)\s+\(?(0x[0-9A-Fa-f]+|\d+)u?\)?", hdr)}
    shared = [k for k in defs if hasattr(eq, k)]
    assert {"EQ_CODEC_PAIR_G", "EQ_CHUNK_INTERLEAVED", "EQ_OUT_BF16", "EQ_FMT_INT8"} <= set(shared)
    for k in shared:
        assert getattr(eq, k) == defs[k], k
