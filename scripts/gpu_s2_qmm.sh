# Config 4 (decode fused into the tcgen05 GEMM) with R18 streams: the value-table decoder
# (default) vs the codes decoder (qa_novals.so), parity tests, and one ncu capture per batch.
OUT=gpurun_out/${TAG:-s2qmm}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -1 $OUT/tests.log
EQ_LIB=$PWD/paper_2601_22787_b200/qa_novals.so timeout 1200 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py -q -x -k "3 or r18" > $OUT/tests_novals.log 2>&1; echo tests_novals=$?; tail -1 $OUT/tests_novals.log
for so in libentquant.so qa_novals.so; do
  for cs in 4096 2048; do
    EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python scripts/bench_qmatmul.py --codec pairg --cs $cs > $OUT/qmm_${so}_$cs.json 2> $OUT/qmm_${so}_$cs.err
    python -c "import json; d=json.load(open('$OUT/qmm_${so}_$cs.json')); print('$so cs=$cs', 'b1', round(d['batch1']['fused_group_ms'],4), round(d['batch1']['fused_group_decode_Tsym_per_s'],3), 'b64', round(d['batch64']['fused_group_ms'],4), round(d['batch64']['fused_group_decode_Tsym_per_s'],3), 'dense', round(d['batch1']['dense_bf16_cublas_ms'],4), 'dec+cublas', round(d['batch1']['decode_then_cublas_ms'],4), 'bits', round(d['effective_bits'],4))"
  done
done
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_qmm_ws -c 4 --csv \
    python scripts/bench_qmatmul.py --codec pairg --cs 4096 --profile > $OUT/ncu_qmm.csv 2> $OUT/ncu_qmm.err; echo ncu=$?
grep -E "k_qmm_ws" $OUT/ncu_qmm.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -20
