# Fused GEMM with 2 row tiles (8 decoder warps) per CTA vs 1: tests and timing at chunks of 4096
# and 2048, then ncu of the better one.
OUT=gpurun_out/${TAG:-s1nt}; mkdir -p $OUT
QVARIANTS="qn1.so qn2.so" TAG=${TAG:-s1nt} bash scripts/gpu_s1_qmm.sh
EQ_LIB=$PWD/paper_2601_22787_b200/qn2.so ncu --set full --clock-control none -k regex:k_qmm_ws -c 2 -o $OUT/qmm_qn2 \
    python scripts/bench_qmatmul.py --profile --cs 2048 > $OUT/qmm_ncu_qn2.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py $OUT/qmm_qn2.ncu-rep > $OUT/qmm_qn2_summary.json 2>&1
