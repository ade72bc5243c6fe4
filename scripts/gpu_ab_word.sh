# A/B of word-decoder variants: word-codec parity tests + a short bench line per .so
for so in ${VARIANTS}; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python -m pytest tests/test_gpu_word_codec.py -x -q > gpurun_out/abw_test_$so.log 2>&1
  t=$?
  EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --lam 230.2 --codec word ${BENCH_ARGS} > gpurun_out/abw_$so.log 2>&1
  echo "$so tests=$t $(python -c "import json,sys; d=json.loads(open('gpurun_out/abw_$so.log').read().strip().splitlines()[-1]); print(round(d['value'],1), 'GB/s', round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1))")"
done
