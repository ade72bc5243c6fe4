"""Host logic of bench.py (no GPU): the chunk-length rule of DESIGN.md §15 and the ncu-capture
matching that ties a committed traffic figure to one kernel source and launch."""
import json
import os
import types

import bench

LANES = 5 * 256 * 148            # k_decode_p: 5 CTAs of 256 lanes on each of 148 SMs


def _args(model="llama-3-8b", mode="interleaved"):
    return types.SimpleNamespace(chunk_symbols=0, model=model, chunk_mode=mode)


def _steps(args, blocks, cs):
    import eqsynth
    shapes = list(eqsynth.block_shapes(args.model)) * blocks
    n = sum((r * c + cs - 1) // cs for r, c in shapes)
    return -(-n // LANES) * cs


def test_chunk_rule_removes_small_partial_rounds_only():
    """4608-symbol chunks only where they remove a last 4096-symbol round that is ≤ ¼ full for a
    share of 1–3 rounds (the measured cases of DESIGN.md §15); 4096 everywhere else; never below
    4096 (the 1.02 × n·Ĥ rate bound)."""
    for model, blocks, want in [("llama-3-8b", 32, 4096), ("llama-3-8b", 16, 4096), ("llama-3-8b", 8, 4608),
                                ("llama-3-8b", 4, 4608), ("llama-3.2-1b", 16, 4096), ("llama-3-70b", 10, 4096),
                                ("llama-3-8b", 1, 4096)]:
        a = _args(model)
        cs = bench.choose_chunk(a, list(range(blocks)), LANES)
        assert cs == want, (model, blocks, cs)
        if cs == 4608:                             # a whole round fewer than 4096 needs
            assert _steps(a, blocks, 4608) // 4608 < _steps(a, blocks, 4096) // 4096


def test_chunk_rule_respects_an_explicit_length():
    a = _args()
    a.chunk_symbols = 2048
    assert bench.choose_chunk(a, list(range(32)), LANES) == 2048


def test_traffic_capture_is_tied_to_kernel_launch_and_layout(tmp_path, monkeypatch):
    """A committed ncu figure is reported only for the same decoder source (sha), block count,
    chunk length and chunk layout — never a stale one."""
    summ = {"pairg": {"kernel_sha": bench.decoder_source_sha(), "blocks": 32, "chunk_symbols": 4096,
                      "chunk_mode": "interleaved", "when": "t", "source": "s",
                      "bf16": {"dram_bytes_per_launch": 1.5e10, "warp_inst_per_launch": 2.0e9}}}
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "ncu_decode_summary.json").write_text(json.dumps(summ))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "decoder_source_sha", lambda: summ["pairg"]["kernel_sha"])
    assert bench.traffic_from_profiles("pairg", "bf16", 32, 4096, "interleaved")[0] == 1.5e10
    assert bench.inst_from_profiles("pairg", "bf16", 32, 4096, "interleaved") == 2.0e9
    assert bench.traffic_from_profiles("pairg", "bf16", 32, 4096, "layer")[0] is None
    assert bench.traffic_from_profiles("pairg", "bf16", 16, 4096, "interleaved")[0] is None
    assert bench.traffic_from_profiles("pairg", "bf16", 32, 4608, "interleaved")[0] is None
    assert bench.traffic_from_profiles("pair", "bf16", 32, 4096, "interleaved")[0] is None
    monkeypatch.setattr(bench, "decoder_source_sha", lambda: "0000000000000000")
    assert bench.traffic_from_profiles("pairg", "bf16", 32, 4096, "interleaved")[0] is None
