# A/B: parity tests on the default build, then short bench lines for each variant .so
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for so in ${VARIANTS}; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --lam 230.2 ${BENCH_ARGS} > gpurun_out/ab_$so.log 2>&1
  echo "$so $(python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$so.log').read().strip().splitlines()[-1]); print(round(d['value'],1), 'GB/s', round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1))")"
done
