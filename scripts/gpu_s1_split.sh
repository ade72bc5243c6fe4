# Escape code out of line per 8 pair steps (EQ_PAIR_SPLIT / EQ_QMM_SPLIT): stand-alone decoder
# and fused GEMM, against the same build without it.
OUT=gpurun_out/${TAG:-s1split}; mkdir -p $OUT
EQ_LIB=$PWD/paper_2601_22787_b200/ab_split.so timeout 1500 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py -q -x > $OUT/tests_split.log 2>&1; echo tests_split=$?; tail -1 $OUT/tests_split.log
VARIANTS="ab_nosplit.so ab_split.so" NCU=1 TAG=${TAG:-s1split} bash scripts/gpu_ab_r2.sh
QVARIANTS="ab_nosplit.so ab_split.so" TAG=${TAG:-s1split} bash scripts/gpu_s1_qmm.sh
