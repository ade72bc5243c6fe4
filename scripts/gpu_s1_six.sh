# 6-CTA build for short launches: tests, per-rank shares (row chunks of 4096, the bench default),
# the 4-block share with layer chunks of 4608 for comparison, and the full set (must stay 5-CTA).
OUT=gpurun_out/${TAG:-s1six}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_pair_codec.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -2 $OUT/tests.log
for spec in "0/8 row 0" "0/4 row 0" "0/2 row 0" "0/8 layer 4608" "0/8 layer 0" "0/1 row 0"; do
  set -- $spec
  tag=$(echo $1 | tr / _)_$2_$3
  timeout 900 python bench.py --as-rank $1 --chunk-mode $2 --chunk-symbols $3 --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/share_$tag.json 2> $OUT/share_$tag.err
  python -c "import json; d=json.loads(open('$OUT/share_$tag.json').read().strip().splitlines()[-1]); s=d.get('per_rank_share') or {}; print('share $1 $2 cs', d['config']['chunk_symbols'], round(d['value'],1), 'GB/s frac', round(d['roofline']['frac'],4), 'bits', round(d['bits_per_param'],4), 'rounds', round(s.get('rounds',0),3), 'ms', round(d['ms_per_step'],4), d['clocks']['reasons'])"
done
