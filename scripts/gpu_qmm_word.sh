# fused decode->tcgen05 GEMM with both codecs: parity tests + config-4 timings
timeout 900 python -m pytest tests/test_gpu_qmatmul.py -x -q > gpurun_out/qmm_test.log 2>&1; echo tests=$?; tail -2 gpurun_out/qmm_test.log
for codec in word byte; do for cs in 2048 1024; do
  timeout 600 python scripts/bench_qmatmul.py --cs $cs --codec $codec > gpurun_out/qmm_${codec}_cs$cs.json 2> gpurun_out/qmm_${codec}_cs$cs.err
  python -c "import json; d=json.load(open('gpurun_out/qmm_${codec}_cs$cs.json')); print('$codec cs=$cs', {k: {kk: round(vv,3) for kk, vv in v.items() if kk.endswith('_ms')} for k, v in d.items() if k.startswith('batch')}, 'bits', round(d['effective_bits'],3))"
done; done
