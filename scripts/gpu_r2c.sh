# Fused GEMM (config 4): parity tests, timing (pair and word codec, row chunks of 4096), and an
# ncu capture of the grouped launch at batch 1 and 64 (tensor pipe, issue, warps).
OUT=gpurun_out/${TAG:-r2c}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -3 $OUT/tests.log
for codec in pair word; do
  timeout 600 python scripts/bench_qmatmul.py --codec $codec > $OUT/qmm_$codec.json 2> $OUT/qmm_$codec.err; echo qmm_$codec=$?
  tail -c 1500 $OUT/qmm_$codec.json
done
ncu --set full --clock-control none --import-source on -k regex:k_qmm_ws -c 2 -o $OUT/qmm \
    python scripts/bench_qmatmul.py --profile > $OUT/qmm_ncu.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py $OUT/qmm.ncu-rep > $OUT/qmm_summary.json 2>&1
for rep in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/bench_$rep.json 2>&1
python -c "import json; d=json.loads(open('$OUT/bench_$rep.json').read().strip().splitlines()[-1]); print('bench', round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d['fp8_out']['value'],1))"
done
