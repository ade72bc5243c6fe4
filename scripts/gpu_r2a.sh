OUT=gpurun_out/r2a; mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo bench=$?
tail -c 4000 $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo ref=$?
tail -c 2000 $OUT/bench_ref.json
TAG=r2a bash scripts/gpu_r2_shares.sh
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x > $OUT/fullsize.log 2>&1; echo fullsize=$?; tail -5 $OUT/fullsize.log
