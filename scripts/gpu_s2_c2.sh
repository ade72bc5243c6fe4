# Config 2 (Llama-3.2-1B set, 1.25 rounds of 4096-symbol chunks): shorter chunks that make whole rounds.
OUT=gpurun_out/${TAG:-s2c2}; mkdir -p $OUT
for cs in 4096 3072 2560 2048; do
  timeout 900 python bench.py --model llama-3.2-1b --chunk-symbols $cs --steps 20 --warmup 3 --no-e2e --no-cpu --no-fp8 > $OUT/c2_$cs.json 2> $OUT/c2_$cs.err
  python -c "import json,sys; d=json.loads(open('$OUT/c2_$cs.json').read().strip().splitlines()[-1]); print('config2', $cs, round(d['value'],1), round(d['roofline']['frac'],4), 'bits', round(d['bits_per_param'],4), 'coded/nH', round(d['rate']['coded_over_nH'],4))"
done
for cs in 3072 2560; do
  timeout 600 python bench.py --as-rank 0/8 --chunk-symbols $cs --steps 20 --warmup 3 --no-e2e --no-cpu --no-fp8 --lam 230.2 > $OUT/g8_$cs.json 2> $OUT/g8_$cs.err
  python -c "import json,sys; d=json.loads(open('$OUT/g8_$cs.json').read().strip().splitlines()[-1]); print('G=8', $cs, round(d['value'],1), round(d['roofline']['frac'],4), 'bits', round(d['bits_per_param'],4), 'coded/nH', round(d['rate']['coded_over_nH'],4), 'rounds', round(d['per_rank_share']['rounds'],3))"
done
