set -x
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --cpu-seconds 5 > gpurun_out/bench1.log 2>&1; echo bench=$?
tail -5 gpurun_out/bench1.log
cat gpurun_out/smoke.log | tail -5
