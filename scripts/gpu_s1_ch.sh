# Dual-chain fused GEMM (EQ_QMM_CH = 2) vs one chain per lane, and the column-by-column chunk
# order of row-chunked layers (EQ_ROW_PERM) in the stand-alone decoders.
OUT=gpurun_out/${TAG:-s1ch}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py tests/test_gpu_pair_codec.py tests/test_gpu_word_codec.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -2 $OUT/tests.log
QVARIANTS="qa_ch1.so libentquant.so" TAG=${TAG:-s1ch} bash scripts/gpu_s1_qmm.sh
for so in ab_noperm.so libentquant.so; do for mode in row layer; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 900 python bench.py --chunk-mode $mode --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/bench_${so}_${mode}.json 2> $OUT/bench_${so}_${mode}.err
  python -c "import json; d=json.loads(open('$OUT/bench_${so}_${mode}.json').read().strip().splitlines()[-1]); print('$so $mode', round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d['fp8_out']['value'],1), d['clocks']['reasons'])"
done; done
