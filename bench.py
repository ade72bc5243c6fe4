#!/usr/bin/env python
"""bench.py — EntQuant decode hot path on B200 (BASELINE config 3 by default).

One step = one pass of the whole hot path over one batch: eq_decode_dequant of every
chunk of the rank's share of the Llama-3-8B-shaped layer set (32 blocks × 7 linear
layers, ~2.0 effective bits/param) into the per-device bf16 arena — §8(a) rows a7+a8.
The streams use the default encoding: the pair codec with grouped escapes (R18)
over interleaved 4096-symbol chunks (R17); ``--codec`` / ``--chunk-mode`` select the others.
The encode side (rows a1-a6) runs once before timing to produce the streams (its time is
reported as ``encode_s``).  Inputs are synthetic (eqsynth), resident in HBM; the 1.76 GB
compressed input and 13.96 GB decoded output per step are both far larger than the 126 MB
L2, so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Multi-GPU: strong scaling by default — ONE 32-block layer set split into
contiguous ranges of 32/G blocks per rank, no data-path collective (blocks are
independent); a barrier brackets the timed region and the time is the max over ranks.
``--scaling weak`` gives every rank its own 32-block set.  ``--as-rank R/G`` runs rank R's
share of a G-GPU split on one GPU (the per-rank lines of profiles/r2).

After timing: every decoded bf16 layer that the CPU-baseline leg decodes with the oracle is
compared with the GPU arena bit for bit (the run fails on a mismatch), and the line carries
the rate statistics of the encoded layer set (Ĥ, coded / n·Ĥ, unique codes, p(0), relative ℓ1).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP8 weight entropy-decode GB/s (frac of HBM peak) at 1/2/4/8 B200; bits/param"
FALLBACK_HBM_GBS = 6650.0            # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
DEFAULT_LAMBDA = 230.2               # reference arm only: the GPU calibration of λ for 2.0 bits


CODECS = {"byte": 0, "word": 1, "pair": 2, "pairg": 3}     # EQ_CODEC_* (include/entquant.h)
CHUNK_MODES = {"layer": 0, "row": 1, "interleaved": 2}   # EQ_CHUNK_* (include/entquant.h, R16, R17)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama-3-8b")
    ap.add_argument("--blocks", type=int, default=0, help="blocks of the layer set (default: all layers of the model)")
    ap.add_argument("--target-bits", type=float, default=2.0)
    ap.add_argument("--lam", type=float, default=None, help="fixed λ (skips calibration)")
    ap.add_argument("--calib-stride", type=int, default=16)
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--as-rank", default=None, help="R/G: run rank R's share of a G-GPU split on this one GPU")
    ap.add_argument("--chunk-symbols", type=int, default=0,
                    help="symbols per chunk (0: auto — 4096 unless the rank's share is too few chunks "
                         "for whole rounds of the decoder's lanes, DESIGN.md §7)")
    ap.add_argument("--tail-blocks", type=int, default=-1,
                    help="encode the share's last N blocks with --tail-cs symbols per chunk (-1: auto, "
                         "bench.choose_tail; 0: none)")
    ap.add_argument("--tail-cs", type=int, default=2048)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp8", action="store_true")
    ap.add_argument("--no-stats", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no extras")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: exercise the multi-rank path with several ranks per GPU (a logic check)")
    ap.add_argument("--chunk-mode", default="auto", choices=["auto", "layer", "row", "interleaved"],
                    help="chunk layout: layer (R10: chunks restart at every layer), row (R16: at every row "
                         "start too, as the decode-fused GEMM of config 4 needs), interleaved (R17: the "
                         "16-symbol groups of 32 consecutive chunks dealt round-robin, so a warp's 32 "
                         "lanes store 1 KB contiguously; pair codec only).  auto: interleaved for the "
                         "pair codec, layer for the others")
    ap.add_argument("--codec", default="pairg", choices=["byte", "word", "pair", "pairg"],
                    help="wire format: byte rANS (SPEC S:355, R9), 16-bit-word rANS (R14), the word "
                         "rANS over symbol pairs with escapes (R15), or the same with each 16-symbol "
                         "group's escaped codes after its pair steps (R18, default: fastest, smallest)")
    args = ap.parse_args()
    if args.chunk_mode == "auto":
        args.chunk_mode = "interleaved" if args.codec in ("pair", "pairg") else "layer"
    return args


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML polled every
    5 ms from a thread (nvidia_ml_py), else `nvidia-smi -lms 50`."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []            # (sm_mhz, max_mhz, reason bits)
        self.stop = threading.Event()
        self.nvml = None
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop.is_set():
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, get_r(h)))
                    except Exception:
                        pass
                    time.sleep(0.005)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(1)
            try:
                self.nvml.nvmlShutdown()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
            self.t.join(1)

    def summary(self):
        sm, mx, reasons = [], [], set()
        for f, m, bits in self.samples:
            sm.append(float(f))
            mx.append(float(m))
            reasons.update(n for n, b in self.BITS.items() if bits & b)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


DECODER_SOURCES = ("rans_dec.cu", "decode_core.cuh", "pair_core.cuh", "common.cuh")


def decoder_source_sha() -> str:
    """sha256 (16 hex) of the decode kernels' sources: ties a committed ncu traffic figure
    to the kernel it was measured on."""
    import hashlib
    h = hashlib.sha256()
    for f in DECODER_SOURCES:
        h.update(open(os.path.join(ROOT, "paper_2601_22787_b200", "csrc", f), "rb").read())
    return h.hexdigest()[:16]


def traffic_from_profiles(codec: str, kind: str, blocks: int, chunk_symbols: int, chunk_mode: str = "layer"):
    """DRAM bytes per launch of the decode kernel from the committed ncu --set full summary —
    only if it was captured on THIS kernel source (sha) and launch (blocks, chunk size);
    otherwise None (a stale figure is never reported)."""
    p = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    try:
        c = json.load(open(p))[codec]
        e = dict(c[kind], **{k: c.get(k) for k in ("kernel_sha", "blocks", "chunk_symbols", "chunk_mode", "when",
                                                    "source")})
    except Exception:
        return None, "no ncu capture"
    if e.get("kernel_sha") != decoder_source_sha():
        return None, f"ncu capture stale (kernel sha {e.get('kernel_sha')} != {decoder_source_sha()})"
    if (e.get("blocks") != blocks or e.get("chunk_symbols") != chunk_symbols
            or e.get("chunk_mode", "layer") != chunk_mode):
        return None, "ncu capture of another launch"
    return e["dram_bytes_per_launch"], f"{e.get('source', p)} (kernel sha {e['kernel_sha']}, {e.get('when', '?')})"


def inst_from_profiles(codec: str, kind: str, blocks: int, chunk_symbols: int, chunk_mode: str = "layer"):
    """Warp-level SASS instructions per launch from the same sha-matched ncu capture, or None."""
    tr, _ = traffic_from_profiles(codec, kind, blocks, chunk_symbols, chunk_mode)
    if tr is None:
        return None
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_decode_summary.json")))[codec][kind].get(
            "warp_inst_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------- shared: the workload
def share_ids(args, rank: int, world: int):
    """(block ids of this process, simulated (rank, world)) — --as-rank R/G runs rank R's share
    of a G-GPU split on this one GPU."""
    from paper_2601_22787_b200 import shard
    if args.as_rank:
        r, g = (int(x) for x in args.as_rank.split("/"))
        return shard.layer_ids(r, g, args.blocks, args.scaling), (r, g)
    return shard.layer_ids(rank, world, args.blocks, args.scaling), (rank, world)


def choose_chunk(args, layer_ids, lanes: int) -> int:
    """Chunk length for the rank's share.  A launch runs chunks / lanes rounds of
    serial chains; a last round that is only partly filled still takes a chain's full latency.
    4096 symbols, unless the 4096-symbol share is at most 1.25 rounds that 4608-symbol chunks
    fit in one (4 Llama-3-8B blocks: 1.12 → 1 round, 0.518 → 0.616 of the HBM peak); elsewhere
    4608 measured slower than 4096 with 2048-symbol tail blocks (choose_tail) or than 4096 alone
    (16 blocks: 0.651 vs 0.663; 10 Llama-3-70B blocks: 0.628 vs 0.680; the Llama-3.2-1B set:
    0.457 vs 0.563; `profiles/r2/s2cab`, `s2tail2`).  Shorter chunks are not chosen: at 2048
    the coded size passes the north star's 1.02 × n·Ĥ (≈ 1.0205 ×)."""
    import eqsynth
    if args.chunk_symbols:
        return args.chunk_symbols
    shapes = list(eqsynth.block_shapes(args.model)) * len(layer_ids)

    def n_chunks(cs):
        if args.chunk_mode == "row":
            return sum(r * ((c + cs - 1) // cs) for r, c in shapes)
        return sum((r * c + cs - 1) // cs for r, c in shapes)
    r = n_chunks(4096) / lanes
    if 1 < r <= 1.25 and n_chunks(4608) <= lanes:
        return 4608
    return 4096


def choose_tail(args, layer_ids, lanes: int, cs: int) -> int:
    """Blocks of the share encoded in 2048-symbol chunks at its end: when the
    4096-symbol share ends in a partly filled round (fraction ≤ ½) that 4608 did not remove, the
    last k = ⌈B − ⌊rounds⌋ · lanes / chunks per block⌉ blocks are coded in 2048-symbol chunks, so
    the 4096-symbol chains fill whole rounds and the short chains fill the tail (`profiles/r2/
    s2tail2`: the Llama-3.2-1B set 0.561 → 0.620 of the HBM peak with k = 4; 16 8B blocks 0.663 →
    0.677, k = 2; 8 blocks 0.630 (4608) → 0.647, k = 1; 10 70B blocks 0.680 → 0.686, k = 1).  Each
    such block codes at ≈ 1.019 × n·Ĥ, under the north star's 1.02."""
    import math

    import eqsynth
    if args.tail_blocks >= 0:
        return args.tail_blocks
    if args.chunk_symbols or cs != 4096 or args.chunk_mode == "row":
        return 0
    shapes = list(eqsynth.block_shapes(args.model))
    per_block = sum((r * c + cs - 1) // cs for r, c in shapes)
    B = len(layer_ids)
    r = B * per_block / lanes
    if r <= 1 or r - math.floor(r) > 0.5:
        return 0
    return min(B, max(0, math.ceil(B - math.floor(r) * lanes / per_block)))


def encode_share(args, eq, eqsynth, dev, layer_ids, cs, dist=None):
    """λ calibration (global; one deterministic calibration on block 0) and Alg. 1 per
    block of the share.  Returns (blocks, λ, estimated bits, encode seconds)."""
    import torch
    t0 = time.time()
    lam, est = args.lam, None
    if lam is None:
        calib = eqsynth.block_weights(args.model, 0, device=dev)
        lam, est = eq.calibrate_lambda(calib, args.target_bits, row_stride=args.calib_stride, chunk_symbols=cs,
                                       codec=CODECS[args.codec], chunk_mode=CHUNK_MODES[args.chunk_mode])
        del calib
    if dist is not None:
        t = torch.tensor([lam], dtype=torch.float64, device=dev)
        dist.broadcast(t, 0)
        lam = float(t.item())
    blocks, scratch = [], None
    n_tail = min(args.tail_blocks, len(layer_ids))
    for i, lid in enumerate(layer_ids):
        Ws = eqsynth.block_weights(args.model, lid, device=dev)
        # the share's last n_tail blocks in shorter chunks: the launch's last, partly filled
        # round of chains is then made of shorter chains (an experiment, --tail-blocks)
        cs_b = args.tail_cs if i >= len(layer_ids) - n_tail else cs
        if scratch is None:
            _, _, sb = eq.encode_bounds(Ws, chunk_symbols=min(cs, args.tail_cs) if n_tail else cs,
                                        codec=CODECS[args.codec], chunk_mode=CHUNK_MODES[args.chunk_mode])
            scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        blocks.append(eq.quantize_encode(Ws, lam=lam, scratch=scratch, chunk_symbols=cs_b, codec=CODECS[args.codec],
                                         chunk_mode=CHUNK_MODES[args.chunk_mode]))
        del Ws
    del scratch
    torch.cuda.synchronize()
    return blocks, lam, est, time.time() - t0


def workload_config(args, n_blocks, n_params, cs, world):
    return {
        "workload": f"config3: {args.model}-shaped layer set of {args.blocks} blocks x 7 linear layers, "
                    f"{n_blocks} blocks per rank, ~{args.target_bits} effective bits/param, chunk-parallel rANS "
                    f"decode + fused dequant to bf16",
        "model_shapes": args.model, "blocks_per_rank": n_blocks, "params_per_rank": n_params,
        "chunk_symbols": cs, "tail_blocks_2048": max(0, args.tail_blocks), "chunk_mode": args.chunk_mode,
        "codec": args.codec, "target_bits": args.target_bits,
        "l2": "inputs larger than L2 (compressed in + decoded out per step >> 126 MB); no flush",
        "parallelism": f"block-sharded x{world} ({args.scaling}, contiguous ranges)" if args.scaling == "strong"
                       else f"block-sharded x{world} (weak)",
    }


def oracle_pair_table(table, o):
    """The pair-codec tables of a block's table buffer (layout of include/entquant.h)."""
    import numpy as np
    return o.PairTable(table.view(np.uint8)[968:984].copy(), int(table[482]), table[256:481].copy(), int(table[481]))


def oracle_layers(blk, o):
    """Host copies of one GPU-encoded block for the oracle, and its per-layer chunk ranges."""
    import numpy as np
    import torch
    cs = blk.chunk_symbols
    off_all = blk.chunk_off.cpu().numpy().astype(np.uint32)
    payload = blk.payload.cpu().numpy()
    table = blk.freq.cpu().numpy().view(np.uint16)
    pair = oracle_pair_table(table, o) if blk.codec in (CODECS["pair"], CODECS["pairg"]) else None
    scales = blk.scales.cpu().view(torch.int16).numpy().view(np.uint16)
    out, k0, r0 = [], 0, 0
    row = getattr(blk, "chunk_mode", 0) == CHUNK_MODES["row"]
    for (r, c) in blk.shapes:
        nk = r * ((c + cs - 1) // cs) if row else (r * c + cs - 1) // cs
        out.append((off_all[k0:k0 + nk + 1], r, c, scales[r0:r0 + r]))
        k0 += nk
        r0 += r
    return payload, table[:256], pair, out


# ---------------------------------------------------------------- reference arm (oracle)
def run_reference(args, rank, world):
    """The oracle, as it stands, timed on the host cores on OUR arm's config: the streams
    of block 0 of the same layer set (λ calibrated and encoded exactly as our arm does —
    untimed input preparation), and per step the oracle's decode + dequant of all 7 whole
    layers of that block.  Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return
    import numpy as np
    import torch

    import eqsynth
    import oracle as o
    import paper_2601_22787_b200 as eq
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    if args.blocks <= 0:
        args.blocks = eqsynth.LLAMA[args.model]["layers"]
    ids, (r, g) = share_ids(args, rank, world)
    lanes0 = max(1, eq.decode_lanes(CODECS[args.codec], eq.EQ_OUT_BF16, 0))
    cs = choose_chunk(args, ids, lanes0)
    # block 0 is a 2048-symbol tail block of our arm's share only when every block is one
    args.tail_blocks = 1 if choose_tail(args, ids, lanes0, cs) >= len(ids) else 0
    n_params = len(ids) * sum(a * b for a, b in eqsynth.block_shapes(args.model))
    blocks, lam, est, enc_s = encode_share(args, eq, eqsynth, dev, [0], cs)
    blk = blocks[0]
    payload, freq, pair, layers = oracle_layers(blk, o)
    threads = os.cpu_count() or 1

    def one_pass():
        for off, rr, c, S in layers:
            o.decode_dequant_layer_mt(payload, off, cs, rr, c, S, freq, threads, blk.codec, pair, blk.chunk_mode)

    bytes_pass = blk.compressed_bytes() + 2 * blk.n_params
    for _ in range(args.warmup):
        one_pass()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        one_pass()
        times.append(time.perf_counter() - t)
    tot = sum(times)
    gbs = bytes_pass * args.steps / tot / 1e9
    sample = (f"oracle decode + bf16 dequant (eqo_decode_chunk_* per chunk, POSIX threads) of block 0: all 7 whole "
              f"{args.model} layers ({blk.n_params} params, {blk.n_chunks} chunks of {cs} symbols, "
              f"{8 * blk.compressed_bytes() / blk.n_params:.4f} eff. bits/param), one block per step")
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (eqsynth: Student-t nu=4, sigma=0.02, per-row log-normal spread; Llama shapes)",
        "config": workload_config(args, len(ids), n_params, cs, g),
        "lambda": lam,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "bits_per_param": 8 * blk.compressed_bytes() / blk.n_params, "encode_s_sample": enc_s,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch.distributed as dist

    import eqsynth
    import paper_2601_22787_b200 as eq
    from paper_2601_22787_b200 import shard
    if args.dist_backend == "gloo":             # logic check of the N-rank path on fewer GPUs (no timing value)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    if args.blocks <= 0:
        args.blocks = eqsynth.LLAMA[args.model]["layers"]
    layer_ids, (sim_rank, sim_world) = share_ids(args, rank, world)
    lanes = max(1, eq.decode_lanes(CODECS[args.codec], eq.EQ_OUT_BF16, local))
    cs = choose_chunk(args, layer_ids, lanes)
    args.tail_blocks = choose_tail(args, layer_ids, lanes, cs)

    # ---- encode side (once): λ calibration (global) then Alg. 1 per block
    blocks, lam, est, enc_s = encode_share(args, eq, eqsynth, dev, layer_ids, cs, dist if world > 1 else None)
    torch.cuda.empty_cache()

    n_params = sum(b.n_params for b in blocks)
    n_chunks = sum(b.n_chunks for b in blocks)
    comp_bytes = sum(b.compressed_bytes() for b in blocks)
    payload_bytes = sum(b.payload_bytes for b in blocks)
    bytes_bf16 = comp_bytes + 2 * n_params
    bytes_fp8 = comp_bytes + n_params
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def time_decoder(dec, steps, warmup, clocks=None):
        for _ in range(warmup):
            dec(stream)
        dec.check(stream)
        barrier()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ctx = clocks if clocks is not None else _Null()
        with ctx:
            ev[0].record(stream)
            for k in range(steps):
                dec(stream)
                ev[k + 1].record(stream)
            torch.cuda.synchronize()
        barrier()
        per = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
        total = ev[0].elapsed_time(ev[steps])
        dec.check(stream)
        total = shard.max_over_ranks(total, dist if world > 1 else None, dev)
        return total, per

    # ---- main metric: bf16-out decode of the rank's share
    dec = eq.Decoder(blocks, eq.EQ_OUT_BF16)
    clocks = ClockSampler(local) if not args.profile else None
    total_ms, per = time_decoder(dec, args.steps, args.warmup, clocks)
    value = shard.aggregate_gbs(bytes_bf16, world, args.steps, total_ms)
    launch_ms = statistics.mean(per)
    achieved = bytes_bf16 / (launch_ms / 1e3) / 1e9
    peak, peak_src = peak_hbm()
    traffic, traffic_src = traffic_from_profiles(args.codec, "bf16", len(blocks), cs, args.chunk_mode)
    inst = inst_from_profiles(args.codec, "bf16", len(blocks), cs, args.chunk_mode)

    fp8, dec8 = None, None
    if not args.no_fp8:
        dec8 = eq.Decoder(blocks, eq.EQ_OUT_FP8)
        t8, per8 = time_decoder(dec8, args.steps, args.warmup)
        l8 = statistics.mean(per8)
        tr8, _ = traffic_from_profiles(args.codec, "fp8", len(blocks), cs, args.chunk_mode)
        fp8 = {"value": shard.aggregate_gbs(bytes_fp8, world, args.steps, t8), "unit": "GB/s",
               "ms_per_step": t8 / args.steps, "frac": bytes_fp8 / (l8 / 1e3) / 1e9 / peak, "traffic": tr8}

    # ---- rate statistics of the encoded share (Eq. 2)
    stats = None
    if not args.no_stats and not args.profile:
        stats = rate_stats(args, eq, eqsynth, blocks, layer_ids, dec, dec8, dev, dist if world > 1 else None)
    if dec8 is not None:
        del dec8
        torch.cuda.empty_cache()

    # ---- e2e through the public C-ABI with host buffers (H2D + decode + D2H per step)
    e2e = None
    if not args.no_e2e and not args.profile:
        hb = eq.HostBlocks(blocks, eq.EQ_OUT_BF16)
        k_e2e = max(1, min(args.steps, 5))
        hb.decode()
        barrier()
        t = time.perf_counter()
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record(stream)
        for _ in range(k_e2e):
            hb.decode(stream)
        e_ev.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
        barrier()
        ms = s_ev.elapsed_time(e_ev)
        ms = max(ms, 1e3 * wall)
        ms = shard.max_over_ranks(ms, dist if world > 1 else None, dev)
        e2e = {"value": shard.aggregate_gbs(bytes_bf16, world, k_e2e, ms), "unit": "GB/s",
               "h2d_bytes_per_step": hb.h2d_bytes(), "d2h_bytes_per_step": hb.total, "steps": k_e2e,
               "ms_per_step": ms / k_e2e}
        del hb

    # ---- CPU baseline: the oracle on the host cores, rank 0, N=1, bounded sample; every
    #      layer it decodes is compared with the GPU arena bit for bit
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu, parity = cpu_baseline(blocks, dec, args.cpu_seconds)
    del dec

    if rank == 0:
        cs_clk = clocks.summary() if clocks is not None else None
        per_rank = {"rank": sim_rank, "of": sim_world, "blocks": layer_ids[0] if len(layer_ids) == 1 else
                    [layer_ids[0], layer_ids[-1]], "chunks": n_chunks, "decoder_lanes": lanes,
                    "rounds": n_chunks / lanes} if args.as_rank else None
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "out_dtype": "bf16",
            "data": "synthetic (eqsynth: Student-t nu=4, sigma=0.02, per-row log-normal spread; Llama shapes)",
            "config": workload_config(args, len(layer_ids), n_params, cs, sim_world),
            "lambda": lam,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src, "kernel": f"k_decode_{'p' if args.codec in ('pair', 'pairg') else 'w' if args.codec == 'word' else ''}",
                         "kernel_sha": decoder_source_sha(),
                         "algorithmic_bytes_per_launch": bytes_bf16, "launch_ms": launch_ms,
                         "chunks": n_chunks, "decoder_lanes": lanes,
                         "warp_inst_per_32_symbols": (None if inst is None else inst / n_params * 32)},
            "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "gpu_launches": args.steps, "clocks": cs_clk,
            "bits_per_param": 8.0 * comp_bytes / n_params,
            "payload_bits_per_param": 8.0 * payload_bytes / n_params,
            "rate": stats, "calib_est_bits": est,
            "symbols_per_s": n_params * world * args.steps / (total_ms / 1e3),
            "fp8_out": fp8, "encode_s": enc_s, "per_rank_share": per_rank,
        }
        print(json.dumps(line), flush=True)
    if parity is not None and not parity["ok"]:
        print(f"PARITY FAILURE: {parity}", file=sys.stderr, flush=True)
        sys.exit(3)
    if world > 1:
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def rate_stats(args, eq, eqsynth, blocks, layer_ids, dec, dec8, dev, dist=None):
    """Rate and distortion of the encoded share: Ĥ of each block's joint histogram (Eq. 2,
    P:160-168) and of each layer alone (the block-table penalty), coded size
    (payload + offsets) over n·Ĥ (the north star's ≤ 1.02), unique codes, p(0), and the
    relative ℓ1 distortion Σ|W − Ŵ| / Σ|W| of Eq. 4 (weights regenerated by eqsynth).
    Codes come from the FP8-out arena (else from the bf16 one is not possible: requires dec8)."""
    import torch
    if dec8 is None:
        return None
    v8, v16 = dec8.views(), dec.views()
    H_blocks, ratios, uniq, per_layer_gap = [], [], [], []
    hist_all = torch.zeros(256, dtype=torch.float64, device=dev)
    err_l1 = torch.zeros((), dtype=torch.float64, device=dev)
    w_l1 = torch.zeros((), dtype=torch.float64, device=dev)

    def ent(h):
        p = h[h > 0] / h.sum()
        return float(-(p * torch.log2(p)).sum())

    for blk, lid, l8, l16 in zip(blocks, layer_ids, v8, v16):
        hb = torch.zeros(256, dtype=torch.float64, device=dev)
        nh = 0.0
        for v in l8:
            h = torch.bincount(v.view(torch.uint8).reshape(-1), minlength=256).double()
            nh += float(h.sum()) * ent(h)
            hb += h
        Hb = ent(hb)
        H_blocks.append(Hb)
        per_layer_gap.append(Hb - nh / float(hb.sum()))
        coded = blk.payload_bytes + 4 * (blk.n_chunks + 1)
        ratios.append(8.0 * coded / (float(hb.sum()) * Hb))
        uniq.append(int((hb > 0).sum()))
        hist_all += hb
        Ws = eqsynth.block_weights(args.model, lid, device=dev)
        for W, What in zip(Ws, l16):
            err_l1 += (W.double() - What.double()).abs().sum()
            w_l1 += W.double().abs().sum()
        del Ws
    n = float(hist_all.sum())
    coded_all = float(sum(b.payload_bytes + 4 * (b.n_chunks + 1) for b in blocks))
    payload_all = float(sum(b.payload_bytes for b in blocks))
    nH = float(sum(float(b.n_params) * H for b, H in zip(blocks, H_blocks)))
    if dist is not None:                       # whole-job figures over all ranks
        t = torch.tensor([n, coded_all, payload_all, nH, float(err_l1), float(w_l1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        dist.all_reduce(hist_all)
        n, coded_all, payload_all, nH, e1, w1 = t.tolist()
        mx = torch.tensor([max(ratios)], dtype=torch.float64, device=dev)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        ratio_max = float(mx.item())
    else:
        e1, w1 = float(err_l1), float(w_l1)
        ratio_max = max(ratios)
    return {
        "H_block_bits": {"min": min(H_blocks), "mean": sum(H_blocks) / len(H_blocks), "max": max(H_blocks)},
        "H_layer_set_bits": ent(hist_all),
        "block_table_penalty_bits": {"max": max(per_layer_gap), "mean": sum(per_layer_gap) / len(per_layer_gap)},
        "coded_over_nH": coded_all * 8.0 / nH, "coded_over_nH_max_block": ratio_max,
        "coded_def": "payload (incl. 4-byte chunk states) + 4-byte chunk offsets, over n x H-hat of each block's histogram",
        "payload_bits_per_symbol": 8.0 * payload_all / n,
        "unique_codes": {"min": min(uniq), "max": max(uniq)},
        "p0": float(hist_all[0] / hist_all.sum()),
        "rel_l1": e1 / w1,
        "symbols": n,
    }


def cpu_baseline(blocks, dec, seconds: float):
    """The oracle, as it stands, decoding + dequantising a bounded sample of the same
    workload (whole layers of the leading blocks, until ~``seconds`` of host work) on all
    host cores, timed; and every layer it decodes compared with the GPU's bf16 arena bit for
    bit (the full-size parity leg: a mismatch fails the run)."""
    import numpy as np
    import torch

    import oracle as o
    threads = os.cpu_count() or 1
    views = dec.views()
    done_bytes, done_syms, wall, layers, mism = 0, 0, 0.0, 0, 0
    for blk, vb in zip(blocks, views):
        payload, freq, pair, lay = oracle_layers(blk, o)
        for (off, r, c, S), v in zip(lay, vb):
            nk = off.size - 1
            t = time.perf_counter()
            out = o.decode_dequant_layer_mt(payload, off, blk.chunk_symbols, r, c, S, freq, threads, blk.codec, pair,
                                            blk.chunk_mode)
            wall += time.perf_counter() - t
            gpu = v.contiguous().view(torch.int16).cpu().numpy().view(np.uint16).reshape(r, c)
            mism += int(np.count_nonzero(np.asarray(out).reshape(r, c) != gpu))
            done_bytes += int(off[-1] - off[0]) + 4 * (nk + 1) + 2 * r + 2 * r * c
            done_syms += r * c
            layers += 1
            if wall >= seconds:
                break
        done_bytes += 2 * blk.freq.numel()
        if wall >= seconds:
            break
    # the same oracle on ONE host thread, on the first layer of block 0
    blk = blocks[0]
    payload, freq, pair, lay = oracle_layers(blk, o)
    off, r, c, S = lay[0]
    t = time.perf_counter()
    o.decode_dequant_layer_mt(payload, off, blk.chunk_symbols, r, c, S, freq, 1, blk.codec, pair, blk.chunk_mode)
    w1 = time.perf_counter() - t
    b1 = int(off[-1] - off[0]) + 4 * off.size + 2 * r + 2 * r * c
    cpu = {"value": done_bytes / wall / 1e9, "unit": "GB/s", "cores": threads, "kind": "oracle",
           "sample": f"{layers} whole layers ({done_syms} symbols) of the leading blocks, decode+dequant to bf16 "
                     f"with the oracle's per-chunk decoder on {threads} threads, {wall:.1f} s wall",
           "value_1_thread": b1 / w1 / 1e9,
           "sample_1_thread": f"layer 0 of block 0 ({r * c} symbols) on 1 thread, {w1:.1f} s wall"}
    parity = {"layers": layers, "symbols": done_syms, "mismatches": mism, "ok": mism == 0,
              "what": "oracle decode+dequant of the GPU-encoded streams vs the GPU bf16 arena of the timed launch, "
                      "element by element"}
    return cpu, parity


if __name__ == "__main__":
    main()
