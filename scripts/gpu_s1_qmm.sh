# Fused GEMM (config 4) A/B: staging ring 64 vs 128 bytes per decoder lane (EQ_WRING), with the
# narrow pair entries and per-step branching; parity tests per variant, timing (pair codec, row
# chunks of 4096 and 2048), one ncu capture of the default variant's grouped launch.
OUT=gpurun_out/${TAG:-s1qmm}; mkdir -p $OUT
for so in ${QVARIANTS:-qa_r64.so libentquant.so qa_s2.so}; do
  L=$PWD/paper_2601_22787_b200/$so
  EQ_LIB=$L timeout 1200 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py -q -x > $OUT/tests_$so.log 2>&1; echo "$so tests=$?"; tail -2 $OUT/tests_$so.log
  for cs in 4096 2048; do
    EQ_LIB=$L timeout 600 python scripts/bench_qmatmul.py --codec pair --cs $cs > $OUT/qmm_${so}_$cs.json 2> $OUT/qmm_${so}_$cs.err
    python -c "import json; d=json.load(open('$OUT/qmm_${so}_$cs.json')); print('$so cs=$cs', 'b1', round(d['batch1']['fused_group_ms'],4), round(d['batch1']['fused_group_decode_Tsym_per_s'],3), 'dec-only', round(d['batch1']['decode_only_ms'],4), 'b64', round(d['batch64']['fused_group_ms'],4), round(d['batch64']['fused_group_decode_Tsym_per_s'],3), 'dense', round(d['batch1']['dense_bf16_cublas_ms'],4), 'dec+cublas', round(d['batch1']['decode_then_cublas_ms'],4))"
  done
done
if [ -n "$NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_qmm_ws -c 2 -o $OUT/qmm \
    python scripts/bench_qmatmul.py --profile > $OUT/qmm_ncu.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py $OUT/qmm.ncu-rep > $OUT/qmm_summary.json 2>&1
fi
if [ -n "$CONFIGS" ]; then
  TAG=${TAG:-s1qmm} bash -c 'timeout 900 python bench.py --model llama-3.2-1b --steps 20 --warmup 3 --no-e2e > gpurun_out/${TAG}/config2.json 2> gpurun_out/${TAG}/config2.err; echo config2=$?'
  python -c "import json; d=json.loads(open('$OUT/config2.json').read().strip().splitlines()[-1]); print('config2', round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1), 'bits', round(d['bits_per_param'],4), 'encode_s', round(d['encode_s'],1), 'cs', d['config']['chunk_symbols'], 'cpu', d['cpu_baseline']['value'], 'parity', d.get('parity',{}).get('ok'))"
  timeout 1500 python bench.py --model llama-3-70b --as-rank 0/8 --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/config5.json 2> $OUT/config5.err; echo config5=$?
  python -c "import json; d=json.loads(open('$OUT/config5.json').read().strip().splitlines()[-1]); print('config5 share', round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1), 'bits', round(d['bits_per_param'],4), 'encode_s', round(d['encode_s'],1), 'cs', d['config']['chunk_symbols'], d['per_rank_share'])"
  M=sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,sm__cycles_active.avg,sm__cycles_elapsed.avg
  for cs in 4608 4096; do
  ncu --metrics $M --clock-control none -k regex:k_decode_p -c 1 --csv python bench.py --as-rank 0/8 --chunk-symbols $cs --profile --steps 1 --warmup 1 --no-e2e --no-cpu --lam 230.2 > $OUT/ncu_share8_$cs.csv 2> $OUT/ncu_share8_$cs.err
  done
fi
