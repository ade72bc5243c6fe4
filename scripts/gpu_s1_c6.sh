# Pair-table shared-memory diet (u16 cum, pair cum inside the escape table, 452-byte codes
# table: 37,888 B per CTA) and 5 vs 6 CTAs/SM (40 registers) for k_decode_p.
OUT=gpurun_out/${TAG:-s1c6}; mkdir -p $OUT
for so in ab_c5.so ab_c6.so; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so python -c "import paper_2601_22787_b200 as eq; print('$so lanes', eq.decode_lanes(eq.EQ_CODEC_PAIR, eq.EQ_OUT_BF16, 0))"
done
timeout 1500 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py tests/test_gpu_pair_codec.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -2 $OUT/tests.log
VARIANTS="ab_c5.so ab_c6.so" NCU=1 TAG=${TAG:-s1c6} BENCH_ARGS="--chunk-mode layer" bash scripts/gpu_ab_r2.sh
EQ_LIB=$PWD/paper_2601_22787_b200/ab_c6.so timeout 600 python -m pytest tests/test_gpu_pair_codec.py -q -x > $OUT/tests_c6.log 2>&1; echo tests_c6=$?
