# Block pipeline (f2) on the pair codec + the decode-fused forward: parity test and timing.
OUT=gpurun_out/${TAG:-s1pipe}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -2 $OUT/tests.log
for cs in 4096 2048; do
  timeout 1200 python scripts/bench_pipeline.py --codec pair --cs $cs > $OUT/pipeline_pair_cs$cs.json 2> $OUT/pipeline_pair_cs$cs.err; echo pipe_$cs=$?
  tail -c 1500 $OUT/pipeline_pair_cs$cs.json; echo
done
