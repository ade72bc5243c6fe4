# Full GPU suite + smoke + a default bench line on the current tree.
OUT=gpurun_out/${TAG:-s2chk}; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?; tail -1 $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo bench=$?
python -c "import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['traffic'], d['roofline'].get('warp_inst_per_32_symbols'), d['clocks'], d['parity']['mismatches'], d['e2e']['value'], d['fp8_out']['value'])"
