#!/usr/bin/env python
"""bench.py — EntQuant decode hot path on B200 (BASELINE config 3 by default).

One step = one pass of the whole hot path over one batch: eq_decode_dequant of every
chunk of the rank's Llama-3-8B-shaped layer set (32 blocks × 7 linear layers, ~2.0
effective bits/param) into the per-device bf16 arena — §8(a) rows a7+a8.  The encode side
(rows a1-a6) runs once before timing to produce the streams (its time is reported as
``encode_s``).  Inputs are synthetic (eqsynth), resident in HBM; the 1.76 GB compressed
input and 13.96 GB decoded output per step are both far larger than the 126 MB L2, so no
flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Multi-GPU: weak scaling — every rank decodes its own 32-block layer set (distinct layers),
no data-path collective (the work shards by block); a barrier brackets the
timed region and the time is the max over ranks.
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


CODECS = {"byte": 0, "word": 1, "pair": 2}     # EQ_CODEC_* (include/entquant.h)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama-3-8b")
    ap.add_argument("--blocks", type=int, default=0, help="blocks per rank (default: all layers of the model)")
    ap.add_argument("--target-bits", type=float, default=2.0)
    ap.add_argument("--lam", type=float, default=None, help="fixed λ (skips calibration)")
    ap.add_argument("--calib-stride", type=int, default=16)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp8", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no extras")
    ap.add_argument("--codec", default="pair", choices=["byte", "word", "pair"],
                    help="wire format: byte rANS (SPEC S:355, R9), 16-bit-word rANS (R14), or the word "
                         "rANS over symbol pairs with escapes (R15, default: fastest, smallest)")
    return ap.parse_args()


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


def traffic_from_profiles(codec: str, kind: str):
    """dram bytes per launch of the decode kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    try:
        d = json.load(open(p))
        return d[codec][kind]["dram_bytes_per_launch"]
    except Exception:
        return None


# ---------------------------------------------------------------- reference arm (oracle)
def run_reference(args, rank, world):
    if rank != 0:
        return
    import eqsynth as _es
    if args.blocks <= 0:                     # same workload config as our arm
        args.blocks = _es.LLAMA[args.model]["layers"]
    n_params_full = args.blocks * sum(r * c for r, c in _es.block_shapes(args.model))
    import numpy as np

    import eqsynth
    import oracle as o
    lam = args.lam if args.lam is not None else DEFAULT_LAMBDA
    threads = os.cpu_count() or 1
    shapes = eqsynth.block_shapes(args.model)
    rows_per = 16
    layers, full_shapes = [], []
    for m, (r, c) in enumerate(shapes):
        ids = list(range(0, r, max(1, r // rows_per)))[:rows_per]
        layers.append(eqsynth.weights_rows(ids, r, c, seed=0, layer=0, matrix=m))
        full_shapes.append((r, c))
    t0 = time.time()
    blk = o.quantize_encode(layers, lam=lam, codec=CODECS[args.codec])
    enc_s = time.time() - t0
    payload = np.frombuffer(blk.payload + b"\0" * 16, dtype=np.uint8)
    # per-layer chunk ranges of the sample block
    sym0, ns = o.chunk_table(blk.layer_shapes, blk.chunk_symbols)
    per_layer, k = [], 0
    for (r, c), S in zip(blk.layer_shapes, blk.scales):
        nk = (r * c + blk.chunk_symbols - 1) // blk.chunk_symbols
        per_layer.append((blk.chunk_off[k:k + nk + 1].copy(), r, c, S))
        k += nk

    def one_pass():
        for off, r, c, S in per_layer:
            o.decode_dequant_layer_mt(payload, off, blk.chunk_symbols, r, c, S, blk.freq, threads, blk.codec, blk.pair)

    t = time.time()
    one_pass()
    once = max(time.time() - t, 1e-4)
    reps = max(1, int(min(3.0, 180.0 / max(1, args.steps + args.warmup)) / once))
    bytes_pass = blk.n_params * 2 + len(blk.payload) + 4 * (blk.n_chunks + 1) + 2 * sum(r for r, _ in blk.layer_shapes) + 512
    for _ in range(args.warmup):
        for _ in range(reps):
            one_pass()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        for _ in range(reps):
            one_pass()
        times.append(time.perf_counter() - t)
    tot = sum(times)
    gbs = bytes_pass * reps * args.steps / tot / 1e9
    sample = (f"oracle decode+dequant (eqo_decode_chunk + bf16 RNE dequant) of {rows_per} rows of each of the 7 "
              f"{args.model} block-0 matrices ({blk.n_params} params, {blk.n_chunks} chunks, λ={lam}, "
              f"{blk.effective_bits():.3f} eff. bits/param), x{reps} per step")
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(args, n_params_full, lam),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "bits_per_param": blk.effective_bits(), "encode_s_sample": enc_s,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n_params, lam):
    return {
        "workload": f"config3: {args.model}-shaped layer set, {args.blocks or 'all'} blocks x 7 linear layers per rank, "
                    f"~{args.target_bits} effective bits/param, chunk-parallel rANS decode + fused dequant to bf16",
        "model_shapes": args.model, "blocks_per_rank": args.blocks, "params_per_rank": n_params,
        "chunk_symbols": 4096, "codec": args.codec, "lambda": lam, "target_bits": args.target_bits,
        "l2": "inputs larger than L2 (compressed in + decoded out per step >> 126 MB); no flush",
        "parallelism": f"block-sharded x{args.gpus} ({args.scaling})",
    }


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
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = eqsynth.LLAMA[args.model]["layers"]
    if args.blocks <= 0:
        args.blocks = L
    from paper_2601_22787_b200 import shard
    layer_ids = shard.layer_ids(rank, world, args.blocks, args.scaling)

    # ---- encode side (once): λ calibration (global) then Alg. 1 per block
    t0 = time.time()
    lam = args.lam
    est = None
    if lam is None:
        calib = eqsynth.block_weights(args.model, 0, device=dev)
        lam, est = eq.calibrate_lambda(calib, args.target_bits, row_stride=args.calib_stride)
        del calib
    if world > 1:
        t = torch.tensor([lam], dtype=torch.float64, device=dev)
        dist.broadcast(t, 0)
        lam = float(t.item())
    blocks = []
    scratch = None
    for lid in layer_ids:
        Ws = eqsynth.block_weights(args.model, lid, device=dev)
        if scratch is None:
            _, _, sb = eq.encode_bounds(Ws)
            scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        blocks.append(eq.quantize_encode(Ws, lam=lam, scratch=scratch, codec=CODECS[args.codec]))
        del Ws
    del scratch
    torch.cuda.synchronize()
    enc_s = time.time() - t0
    torch.cuda.empty_cache()

    n_params = sum(b.n_params for b in blocks)
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

    # ---- main metric: bf16-out decode of the whole layer set
    dec = eq.Decoder(blocks, eq.EQ_OUT_BF16)
    clocks = ClockSampler(local) if not args.profile else None
    total_ms, per = time_decoder(dec, args.steps, args.warmup, clocks)
    value = shard.aggregate_gbs(bytes_bf16, world, args.steps, total_ms)
    launch_ms = statistics.mean(per)
    achieved = bytes_bf16 / (launch_ms / 1e3) / 1e9
    peak, peak_src = peak_hbm()

    fp8 = None
    if not args.no_fp8:
        del dec
        torch.cuda.empty_cache()
        dec8 = eq.Decoder(blocks, eq.EQ_OUT_FP8)
        t8, per8 = time_decoder(dec8, args.steps, args.warmup)
        l8 = statistics.mean(per8)
        fp8 = {"value": shard.aggregate_gbs(bytes_fp8, world, args.steps, t8), "unit": "GB/s",
               "ms_per_step": t8 / args.steps, "frac": bytes_fp8 / (l8 / 1e3) / 1e9 / peak,
               "traffic": traffic_from_profiles(args.codec, "fp8")}
        del dec8
        torch.cuda.empty_cache()
    else:
        del dec

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

    # ---- CPU baseline: the oracle on the host cores, rank 0, N=1, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu = cpu_baseline(blocks, args.cpu_seconds)

    if rank == 0:
        cs = clocks.summary() if clocks is not None else None
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "out_dtype": "bf16",
            "data": "synthetic (eqsynth: Student-t nu=4, sigma=0.02, per-row log-normal spread; Llama shapes)",
            "config": workload_config(args, n_params, lam),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profiles(args.codec, "bf16"),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": bytes_bf16, "launch_ms": launch_ms},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps, "clocks": cs,
            "bits_per_param": 8.0 * comp_bytes / n_params,
            "payload_bits_per_param": 8.0 * payload_bytes / n_params,
            "calib_est_bits": est, "symbols_per_s": n_params * world * args.steps / (total_ms / 1e3),
            "fp8_out": fp8, "encode_s": enc_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def cpu_baseline(blocks, seconds: float):
    """The oracle, as it stands, decoding+dequantising a bounded sample of the same
    workload (whole layers of the leading blocks, until ~``seconds`` of host work) on all
    host cores.  Timing only — not a parity check."""
    import numpy as np
    import torch

    import oracle as o
    threads = os.cpu_count() or 1
    done_bytes, done_syms, wall, layers = 0, 0, 0.0, 0
    for blk in blocks:
        cs = blk.chunk_symbols
        off_all = blk.chunk_off.cpu().numpy().astype(np.uint32)
        payload = blk.payload.cpu().numpy()
        table = blk.freq.cpu().numpy().view(np.uint16)
        freq = table[:256]
        pair = None
        if blk.codec == CODECS["pair"]:                    # the table buffer layout of include/entquant.h
            pair = o.PairTable(table.view(np.uint8)[968:984].copy(), int(table[482]), table[256:481].copy(),
                               int(table[481]))
        scales = blk.scales.cpu().view(torch.int16).numpy().view(np.uint16)
        k0, r0 = 0, 0
        for (r, c) in blk.shapes:
            nk = (r * c + cs - 1) // cs
            off = off_all[k0:k0 + nk + 1]
            t = time.perf_counter()
            o.decode_dequant_layer_mt(payload, off, cs, r, c, scales[r0:r0 + r], freq, threads, blk.codec, pair)
            wall += time.perf_counter() - t
            done_bytes += int(off[-1] - off[0]) + 4 * (nk + 1) + 2 * r + 2 * r * c
            done_syms += r * c
            layers += 1
            k0 += nk
            r0 += r
            if wall >= seconds:
                break
        done_bytes += 512
        if wall >= seconds:
            break
    # the same oracle on ONE host thread, on the first layer of block 0
    blk = blocks[0]
    r, c = blk.shapes[0]
    nk = (r * c + blk.chunk_symbols - 1) // blk.chunk_symbols
    off = blk.chunk_off.cpu().numpy().astype(np.uint32)[:nk + 1]
    t = time.perf_counter()
    table = blk.freq.cpu().numpy().view(np.uint16)
    pair = None
    if blk.codec == CODECS["pair"]:
        pair = o.PairTable(table.view(np.uint8)[968:984].copy(), int(table[482]), table[256:481].copy(), int(table[481]))
    o.decode_dequant_layer_mt(blk.payload.cpu().numpy(), off, blk.chunk_symbols, r, c,
                              blk.scales.cpu().view(torch.int16).numpy().view(np.uint16)[:r],
                              table[:256], 1, blk.codec, pair)
    w1 = time.perf_counter() - t
    b1 = int(off[-1] - off[0]) + 4 * (nk + 1) + 2 * r + 2 * r * c
    return {"value": done_bytes / wall / 1e9, "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"{layers} whole layers ({done_syms} symbols) of the leading blocks, decode+dequant to bf16 "
                      f"with eqo_decode_chunk on {threads} threads, {wall:.1f} s wall",
            "value_1_thread": b1 / w1 / 1e9,
            "sample_1_thread": f"layer 0 of block 0 ({r * c} symbols) on 1 thread, {w1:.1f} s wall"}


if __name__ == "__main__":
    main()
