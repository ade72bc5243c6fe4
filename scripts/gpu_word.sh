# word-codec bring-up: all GPU parity tests, then byte vs word (ring 128 / 64) bench lines
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for cfg in "byte libentquant.so" "word libentquant.so" "word libentquant_r64.so"; do
  set -- $cfg
  EQ_LIB=$PWD/paper_2601_22787_b200/$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --lam 230.2 --codec $1 > gpurun_out/ab_$1_$2.log 2>&1
  echo "$1 $2 $(python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$1_$2.log').read().strip().splitlines()[-1]); print(round(d['value'],1), 'GB/s', round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1), 'bits', round(d['bits_per_param'],4))")"
done
