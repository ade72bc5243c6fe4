# Full GPU test suite + smoke + bench in both chunk modes (R16 row chunking vs R10 layer chunking).
OUT=gpurun_out/${TAG:-s1chk}; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?; tail -1 $OUT/smoke.log
for mode in row layer; do for rep in 1 2; do
  timeout 900 python bench.py --chunk-mode $mode --steps 20 --warmup 3 --no-e2e --no-cpu > $OUT/bench_${mode}_$rep.json 2> $OUT/bench_${mode}_$rep.err
  python -c "import json; d=json.loads(open('$OUT/bench_${mode}_$rep.json').read().strip().splitlines()[-1]); print('$mode', round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d['fp8_out']['value'],1), 'bits', round(d['bits_per_param'],4), 'coded/nH', round(d['rate']['coded_over_nH'],4), 'enc', round(d['encode_s'],1), d['clocks']['reasons'])"
done; done
