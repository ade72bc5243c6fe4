# CTAs/SM (wave quantisation) experiment on the 32-block bench
for occ in 6 5 4; do
  EQ_DECW_OCC=$occ timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --lam 230.2 > gpurun_out/occ_$occ.log 2>&1
  echo "occ=$occ $(python -c "import json; d=json.loads(open('gpurun_out/occ_$occ.log').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1))")"
done
for b in 24 28; do
  for occ in 6 5; do
  EQ_DECW_OCC=$occ timeout 600 python bench.py --blocks $b --steps 10 --warmup 3 --no-e2e --no-cpu --lam 230.2 > gpurun_out/occb_$occ.log 2>&1
  echo "blocks=$b occ=$occ $(python -c "import json; d=json.loads(open('gpurun_out/occb_$occ.log').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1))")"
  done
done
