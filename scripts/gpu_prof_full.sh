# one ncu --set full capture of the decode kernels (bf16 and fp8), 8 blocks
set -x
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:k_decode -s ${SKIP:-1} -c ${COUNT:-2} -o $OUT/decode \
    python bench.py --profile --blocks ${PBLOCKS:-8} --steps 1 --warmup 1 --no-e2e --no-cpu --lam ${LAM:-230.2} > $OUT/full_bench.log 2>&1
echo full=$?
python scripts/ncu_summary.py $OUT/decode.ncu-rep > $OUT/summary.json 2>&1
head -c 3000 $OUT/summary.json
