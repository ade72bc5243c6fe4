"""Condense an `ncu --metrics ... --csv` log (one row per kernel x metric) into one line per
launch: kernel, time, instructions per decoded symbol, issue/warps active, shared wavefronts
and bank conflicts per symbol, DRAM bytes.  usage: python scripts/ncu_csv_summary.py f.csv [symbols]"""
import csv
import io
import sys

SYMS = 6979321856          # Llama-3-8B layer set (config 3), one bench launch


def main(path, syms=SYMS):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    k_id, k_name, k_m, k_u, k_v = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    launches = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        d = launches.setdefault(r[k_id], {"kernel": r[k_name][:40]})
        try:
            d[r[k_m]] = float(r[k_v].replace(",", ""))
        except ValueError:
            d[r[k_m]] = r[k_v]
    for lid, d in launches.items():
        ins = d.get("sm__inst_executed.sum", 0)
        wf = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 0)
        bc = d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 0)
        print(f"{lid} {d['kernel']}: t={d.get('gpu__time_duration.sum', 0)/1e6:.3f} ms  "
              f"warp-instr/32sym={32*ins/syms:.2f}  issue={d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f}%  "
              f"warps={d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f}%  "
              f"smem-wf/32sym={32*wf/syms:.2f} conflicts={bc/max(wf,1):.2f}  "
              f"alu={d.get('sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 0):.1f}% "
              f"lsu={d.get('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 0):.1f}% "
              f"fma={d.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 0):.1f}%  "
              f"dram={(d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0))/1e9:.2f} GB  "
              f"lanes/instr={d.get('smsp__thread_inst_executed_per_inst_executed.ratio', 0):.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else SYMS)
