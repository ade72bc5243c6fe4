# A/B of decoder variants: word parity tests, bench line and DRAM bytes (ncu, one pass) per .so
for so in ${VARIANTS}; do
  export EQ_LIB=$PWD/paper_2601_22787_b200/$so
  timeout 600 python -m pytest tests/test_gpu_word_codec.py -x -q > gpurun_out/abd_test_$so.log 2>&1; t=$?
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --lam 230.2 ${BENCH_ARGS} > gpurun_out/abd_$so.log 2>&1
  echo "$so tests=$t $(python -c "import json; d=json.loads(open('gpurun_out/abd_$so.log').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1))")"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_decode -c 2 --csv python bench.py --profile --steps 1 --warmup 0 --no-e2e --no-cpu --lam 230.2 ${BENCH_ARGS} 2>/dev/null | grep -E '"(dram|gpu__time)' | awk -F'","' '{print "   ", $5, $(NF-2), $NF}'
done
