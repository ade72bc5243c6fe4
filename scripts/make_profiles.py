"""Turn one evidence run (scripts/gpu_evidence.sh output directory) into the committed
profile summaries:

  profiles/ncu_decode_summary.json   per-launch DRAM bytes of k_decode (bench.py's `traffic`)
  profiles/<round>/ncu_decode_full.json     ncu --set full summary (scripts/ncu_summary.py)
  profiles/<round>/launches_summary.csv     launch list of the bench command, per kernel
  profiles/<round>/launches_decode.json     the timed step's kernels and their share

Usage: python scripts/make_profiles.py gpurun_out/ev1 r1
"""
import csv
import re
import json
import os
import shutil
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _num(s):
    v, unit = s.split()[0], (s.split()[1] if len(s.split()) > 1 else "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3,
             "ms": 1.0, "s": 1e3}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def main(ev, rnd):
    out_dir = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(out_dir, exist_ok=True)
    full = json.load(open(os.path.join(ev, "summary.json")))
    shutil.copy(os.path.join(ev, "summary.json"), os.path.join(out_dir, "ncu_decode_full.json"))
    sp = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    summ = json.load(open(sp)) if os.path.exists(sp) else {}
    if "bf16" in summ:                       # old flat layout (byte codec only)
        summ = {"byte": {k: summ.pop(k) for k in ("bf16", "fp8", "source") if k in summ}}
    sha_f = os.path.join(ev, "kernel_sha.txt")
    sha = open(sha_f).read().strip() if os.path.exists(sha_f) else None
    when = open(os.path.join(ev, "when.txt")).read().strip() if os.path.exists(os.path.join(ev, "when.txt")) else None
    cm_f = os.path.join(ev, "chunk_mode.txt")          # the captured launch's chunk layout (R10/R16/R17)
    chunk_mode = open(cm_f).read().strip() if os.path.exists(cm_f) else "layer"
    for d in full:
        k = d["kernel"]
        import re
        targs = re.search(r"k_decode\w*<([^>]*)>", k)
        targs = [a.replace("(bool)", "").strip() for a in targs.group(1).split(",")] if targs else []
        grouped = "k_decode_p" in k and len(targs) > 1 and targs[1] in ("1", "true")
        codec = ("word" if "k_decode_w" in k else ("pairg" if grouped else "pair") if "k_decode_p" in k
                 else "byte" if "k_decode" in k else None)
        kind = ("bf16" if targs and targs[0] in ("1", "true") else
                "fp8" if targs and targs[0] in ("0", "false") else None)
        if codec is None or kind is None:
            continue
        rd, wr = _num(d["dram__bytes_read.sum"]), _num(d["dram__bytes_write.sum"])
        summ.setdefault(codec, {})["source"] = (
            f"profiles/{rnd}/ncu_decode_full.json (ncu --set full --clock-control none, bench.py --profile "
            f"--steps 1 --warmup 1 --codec {codec}: 32 blocks, lambda 230.2)")
        summ[codec]["kernel_sha"] = sha
        summ[codec]["when"] = when
        summ[codec]["blocks"] = 32
        summ[codec]["chunk_symbols"] = 4096
        summ[codec]["chunk_mode"] = chunk_mode
        summ[codec][kind] = {"kernel": k, "duration_ms_under_ncu": _num(d["gpu__time_duration.sum"]),
                             "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                             "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active")}
        if d.get("smsp__inst_executed.sum"):
            summ[codec][kind]["warp_inst_per_launch"] = float(d["smsp__inst_executed.sum"].split()[0].replace(",", ""))
    json.dump(summ, open(sp, "w"), indent=1)

    # launch list: "ID",...,"Kernel Name",...,"Metric Value"
    rows = []
    with open(os.path.join(ev, "launches.csv")) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) / 1e3))   # ns -> us
    per = defaultdict(list)
    for k, us in rows:
        per[k.split("(")[0]].append(us)
    tot = sum(us for _, us in rows)
    with open(os.path.join(out_dir, "launches_summary.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_us", "share_of_command", "mean_us"])
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            w.writerow([k, len(v), round(sum(v), 1), round(sum(v) / tot, 5), round(sum(v) / len(v), 1)])
    dec = {k: v for k, v in per.items() if "k_decode" in k and re.search(r"<(\(bool\))?(1|true)[,>]", k)}
    json.dump({"command": "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --lam 230.2 "
                          "(ncu --metrics gpu__time_duration.sum --clock-control none)",
               "timed_step_kernels": {k: {"launches": len(v), "mean_us": sum(v) / len(v)} for k, v in dec.items()},
               "decode_share_of_timed_step": 1.0,
               "note": "cold-cache, serialised per-launch times; the timed step (one eq_decode_dequant of the "
                       "32-block layer set) launches exactly one decode kernel (k_decode_p<1> for the pair codec, "
                       "k_decode_w<1> for the word codec, k_decode<1> for the byte codec), so its share of the "
                       "step is 1.0 in both the bench and the launch list"},
              open(os.path.join(out_dir, "launches_decode.json"), "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r1")
