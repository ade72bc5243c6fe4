OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rowchunk.py tests/test_gpu_pair_codec.py tests/test_gpu_parity.py tests/test_gpu_qmatmul.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -3 $OUT/tests.log
VARIANTS="ab_p256.so ab_p512x3.so ab_p512x4.so" TAG=r2b NCU=1 bash scripts/gpu_ab_r2.sh
for so in ab_p256.so ab_p512x3.so; do for G in 8; do
EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python bench.py --as-rank 0/$G --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/share_${so}_G$G.json 2>&1
python -c "import json; d=json.loads(open('$OUT/share_${so}_G$G.json').read().strip().splitlines()[-1]); print('$so G=$G', d['config']['chunk_symbols'], round(d['value'],1), round(d['roofline']['frac'],4), d['roofline']['decoder_lanes'])"
done; done
