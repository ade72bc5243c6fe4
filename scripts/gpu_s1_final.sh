# Final evidence for round 2 (session 2): gpu_evidence.sh (tests, smoke, bench, reference arm,
# launch list, ncu --set full of the bench's decode launch) + the word and byte codecs' lines.
TAG=${TAG:-s1final} bash scripts/gpu_evidence.sh
OUT=gpurun_out/${TAG:-s1final}
for codec in word byte; do
  timeout 900 python bench.py --codec $codec --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats > $OUT/bench_$codec.json 2> $OUT/bench_$codec.err
  python -c "import json; d=json.loads(open('$OUT/bench_$codec.json').read().strip().splitlines()[-1]); print('$codec', round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d['fp8_out']['value'],1), 'bits', round(d['bits_per_param'],4), d['clocks']['reasons'])"
done
timeout 900 python bench.py --chunk-mode row --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats > $OUT/bench_row.json 2> $OUT/bench_row.err
python -c "import json; d=json.loads(open('$OUT/bench_row.json').read().strip().splitlines()[-1]); print('pair row', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['reasons'])"
