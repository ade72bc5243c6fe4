# compute-sanitizer memcheck / racecheck / synccheck on the R18 decoder (grouped escapes, value
# table, escape patch without ring waits) and the R18 fused GEMM.
OUT=gpurun_out/${TAG:-s2san}; mkdir -p $OUT
SEL_DEC='tests/test_gpu_pair_codec.py tests/test_gpu_interleaved.py -k "r18 and (oracle_streams or extreme or runaway or byte_identical)"'
SEL_QMM='tests/test_gpu_rowchunk.py -k "escape_heavy and r18"'
for tool in memcheck racecheck synccheck; do
  for sel in DEC QMM; do
    eval S=\$SEL_$sel
    eval timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $S -q -x -p no:cacheprovider > $OUT/${tool}_$sel.txt 2>&1
    echo "$tool $sel rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $OUT/${tool}_$sel.txt | tr '\n' ' ')"
  done
done
