# ncu evidence for the decode kernel (one GPU; short bench in --profile mode)
set -x
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --profile --blocks ${BLOCKS:-32} --steps 2 --warmup 1 --no-e2e --no-cpu --lam ${LAM:-230.2} > $OUT/launches_bench.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_decode -s ${SKIP:-1} -c ${COUNT:-2} -o $OUT/decode \
    python bench.py --profile --blocks ${PBLOCKS:-8} --steps 1 --warmup 1 --no-e2e --no-cpu --lam ${LAM:-230.2} > $OUT/full_bench.log 2>&1
echo full=$?
ls -la $OUT
