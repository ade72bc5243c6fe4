# compute-sanitizer memcheck / racecheck / synccheck on the round-2 pair decoder (narrow entries,
# shared-memory diet with the pair cum inside the escape table) and the two-tile fused GEMM.
OUT=gpurun_out/${TAG:-s1san}; mkdir -p $OUT
SEL_DEC='tests/test_gpu_pair_codec.py -k "oracle_streams or extreme or runaway"'
SEL_QMM='tests/test_gpu_rowchunk.py -k "qmatmul"'
for tool in memcheck racecheck synccheck; do
  for sel in DEC QMM; do
    eval S=\$SEL_$sel
    eval timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $S -q -x -p no:cacheprovider > $OUT/${tool}_$sel.txt 2>&1
    echo "$tool $sel rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $OUT/${tool}_$sel.txt | tr '\n' ' ')"
  done
done
