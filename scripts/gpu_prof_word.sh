# word-codec decoder: short bench + ncu --set full of k_decode_w (bf16 + fp8), 8 blocks
set -x
OUT=gpurun_out/${TAG:-profw}
mkdir -p $OUT
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --lam 230.2 --codec word > $OUT/bench.log 2>&1
python -c "import json; d=json.loads(open('$OUT/bench.log').read().strip().splitlines()[-1]); print('word', round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode -s ${SKIP:-1} -c ${COUNT:-2} -o $OUT/decode \
    python bench.py --profile --blocks ${PBLOCKS:-8} --steps 1 --warmup 1 --no-e2e --no-cpu --lam 230.2 --codec word > $OUT/full_bench.log 2>&1
echo full=$?
python scripts/ncu_summary.py $OUT/decode.ncu-rep > $OUT/summary.json 2>&1
head -c 4000 $OUT/summary.json
