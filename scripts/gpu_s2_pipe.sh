# Block pipeline (§8(f) row 2) and the decode-fused forward with R18 row-chunked streams.
OUT=gpurun_out/${TAG:-s2pipe}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -2 $OUT/tests.log
for cs in 4096 2048; do
  timeout 1200 python scripts/bench_pipeline.py --codec pairg --cs $cs > $OUT/pipeline_pairg_cs$cs.json 2> $OUT/pipeline_pairg_cs$cs.err; echo pipe_$cs=$?
  tail -c 1500 $OUT/pipeline_pairg_cs$cs.json; echo
done
