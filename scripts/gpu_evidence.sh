# Round evidence on one B200: tests, smoke, default bench (with e2e, cpu baseline + full-size
# parity leg, rate statistics), the reference arm, the ncu launch list of the bench command, and
# one ncu --set full capture of the decode kernels at the bench's launch configuration.
set -x
OUT=gpurun_out/${TAG:-evidence}
mkdir -p $OUT
date -u +%Y-%m-%dT%H:%M:%SZ > $OUT/when.txt
python -c "import bench; print(bench.decoder_source_sha())" > $OUT/kernel_sha.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
if [ -z "$NOTEST" ]; then
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
fi
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/launches_bench.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 1 -c 2 -o $OUT/decode \
    python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu --lam 230.2 > $OUT/full_bench.log 2>&1; echo full=$?
python scripts/ncu_summary.py $OUT/decode.ncu-rep > $OUT/summary.json 2>&1
python -c "import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print(d['config'].get('chunk_mode','layer'))" > $OUT/chunk_mode.txt
tail -c 3000 $OUT/bench.json
