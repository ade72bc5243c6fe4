# Per-rank shares of the §8(e) split measured on one B200 (bench.py --as-rank R/G): G = 2, 4, 8
# (16, 8, 4 Llama-3-8B blocks) at chunk lengths 4096 / 2048 / 1024 and the auto choice.
OUT=gpurun_out/${TAG:-shares}
mkdir -p $OUT
for G in 2 4 8; do
  for cs in ${CSLIST:-4096 2048 1024 0}; do
    timeout 600 python bench.py --as-rank 0/$G --chunk-symbols $cs --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/share_G${G}_cs${cs}.json 2> $OUT/share_G${G}_cs${cs}.err
    python -c "import json; d=json.loads(open('$OUT/share_G${G}_cs${cs}.json').read().strip().splitlines()[-1]); print('G=$G cs=$cs', d['config']['chunk_symbols'], round(d['value'],1), 'GB/s frac', round(d['roofline']['frac'],4), 'bits', round(d['bits_per_param'],4), 'rounds', round(d['per_rank_share']['rounds'],3), 'ms', round(d['ms_per_step'],4))"
  done
done
