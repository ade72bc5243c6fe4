# quick GPU iteration: parity tests + a short bench line
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/bench_quick.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench_quick.log | cut -c1-1500
