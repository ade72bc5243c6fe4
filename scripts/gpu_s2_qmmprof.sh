# ncu --set full of the config-4 fused launch (R18, row chunks of 2048, batch 1 and 64) for the
# per-instruction stall attribution.
OUT=gpurun_out/${TAG:-s2qprof}; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:k_qmm_ws -c 2 -o $OUT/qmm \
    python scripts/bench_qmatmul.py --codec pairg --cs 2048 --profile > $OUT/ncu.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py $OUT/qmm.ncu-rep > $OUT/summary.json 2>&1
python -c "
import json; d=json.load(open('$OUT/summary.json'))
for x in d: print(x['kernel'], x.get('gpu__time_duration.sum'), x.get('smsp__issue_active.avg.pct_of_peak_sustained_active'), x.get('sm__warps_active.avg.pct_of_peak_sustained_active'), x.get('stalls_per_issue'))
"
