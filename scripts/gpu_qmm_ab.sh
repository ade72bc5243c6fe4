# fused GEMM variants: qmatmul parity tests + config-4 timings per .so
for so in ${VARIANTS}; do
  export EQ_LIB=$PWD/paper_2601_22787_b200/$so
  timeout 300 python -m pytest tests/test_gpu_qmatmul.py -x -q > gpurun_out/qab_test_$so.log 2>&1; t=$?
  echo "$so tests=$t $(tail -1 gpurun_out/qab_test_$so.log)"
  if [ $t -eq 0 ]; then
    for cs in 2048 1024; do
      timeout 300 python scripts/bench_qmatmul.py --cs $cs --codec word > gpurun_out/qab_${so}_$cs.json 2>/dev/null
      python -c "import json; d=json.load(open('gpurun_out/qab_${so}_$cs.json')); print('   cs=$cs', {k: {kk: round(vv,3) for kk, vv in v.items() if kk.endswith('_ms') and kk.startswith('fused')} for k, v in d.items() if k.startswith('batch')})"
    done
  fi
done
