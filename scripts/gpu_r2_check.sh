# Round-2 check on one B200: all GPU tests, smoke, one bench line (fixed λ), and one ncu
# --set full capture of the bf16 decode launch of the bench (summarised by ncu_summary.py).
OUT=gpurun_out/${TAG:-check}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --lam 230.2 > $OUT/bench.json 2> $OUT/bench.err; echo bench=$?
tail -c 600 $OUT/bench.json
if [ -n "$FULL" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_decode_p -s 1 -c 1 -o $OUT/decode \
    python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu --no-fp8 --lam 230.2 > $OUT/full_bench.log 2>&1; echo full=$?
python scripts/ncu_summary.py $OUT/decode.ncu-rep > $OUT/summary.json 2>&1
fi
