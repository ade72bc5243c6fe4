# A/B of pair-decoder variants: pair-codec parity tests + a short bench line per .so
for so in ${VARIANTS}; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python -m pytest tests/test_gpu_pair_codec.py -x -q > gpurun_out/abp_test_$so.log 2>&1
  t=$?
  for rep in 1 2; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --codec pair ${BENCH_ARGS} > gpurun_out/abp_${so}_$rep.log 2>&1
  echo "$so rep$rep tests=$t $(python -c "import json,sys; d=json.loads(open('gpurun_out/abp_${so}_$rep.log').read().strip().splitlines()[-1]); print(round(d['value'],1), 'GB/s', round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1))")"
  done
done
