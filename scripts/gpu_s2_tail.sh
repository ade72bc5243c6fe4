# Config 2 (1.25 rounds of 4096-symbol chains): the last k blocks in 2048-symbol chunks.
OUT=gpurun_out/${TAG:-s2tail}; mkdir -p $OUT
for k in 0 2 4 6 8; do
  timeout 900 python bench.py --model llama-3.2-1b --tail-blocks $k --steps 20 --warmup 3 --no-cpu --no-e2e > $OUT/c2_tail$k.json 2> $OUT/c2_tail$k.err
  python -c "import json; d=json.loads(open('$OUT/c2_tail$k.json').read().strip().splitlines()[-1]); print('config2 tail', $k, round(d['value'],1), round(d['roofline']['frac'],4), 'bits', round(d['bits_per_param'],4), 'coded/nH', round(d['rate']['coded_over_nH'],4), 'max block', round(d['rate']['coded_over_nH_max_block'],4))"
done
