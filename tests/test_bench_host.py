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


def test_chunk_rule_and_tail_blocks():
    """4608-symbol chunks only for a share of ≤ 1.25 rounds that they fit in one; otherwise 4096,
    with the share's last k blocks in 2048-symbol chunks when its last round is ≤ ½ full —
    k = ⌈B − ⌊rounds⌋ · lanes / chunks per block⌉ (the measured cases of DESIGN.md §15); the
    32-block config-3 set (9.0 rounds) is plain 4096."""
    for model, blocks, want_cs, want_k in [("llama-3-8b", 32, 4096, 0), ("llama-3-8b", 16, 4096, 2),
                                           ("llama-3-8b", 8, 4096, 1), ("llama-3-8b", 4, 4608, 0),
                                           ("llama-3.2-1b", 16, 4096, 4), ("llama-3-70b", 10, 4096, 1),
                                           ("llama-3-8b", 1, 4096, 0)]:
        a = _args(model)
        a.tail_blocks = -1
        cs = bench.choose_chunk(a, list(range(blocks)), LANES)
        k = bench.choose_tail(a, list(range(blocks)), LANES, cs)
        assert (cs, k) == (want_cs, want_k), (model, blocks, cs, k)
        if k:                                      # the 4096-symbol blocks fill whole rounds
            import eqsynth
            per = sum((r * c + 4095) // 4096 for r, c in eqsynth.block_shapes(model))
            assert (blocks - k) * per <= int(blocks * per / LANES) * LANES
    a = _args()
    a.tail_blocks = 3                              # explicit
    assert bench.choose_tail(a, list(range(16)), LANES, 4096) == 3
    a = _args(mode="row")
    a.tail_blocks = -1
    assert bench.choose_tail(a, list(range(16)), LANES, 4096) == 0      # the fused GEMM's streams stay uniform


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
