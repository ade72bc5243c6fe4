# Run-to-run stability of the headline on one box: five default bench lines (no CPU / e2e legs).
OUT=gpurun_out/${TAG:-s2rep}; mkdir -p $OUT
for i in 1 2 3 4 5; do
  timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  python -c "import json; d=json.loads(open('$OUT/bench_$i.json').read().strip().splitlines()[-1]); print($i, round(d['value'],1), round(d['roofline']['frac'],4), d['roofline']['traffic'], round(d['fp8_out']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['rate']['coded_over_nH'],4))"
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
