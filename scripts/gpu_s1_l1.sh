# Fused GEMM without the escape symbol table when it costs the third CTA per SM (batch 64),
# 512-byte-aligned dynamic window without slack: tests and timing.
OUT=gpurun_out/${TAG:-s1l1}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -2 $OUT/tests.log
QVARIANTS="${QV:-libentquant.so}" TAG=${TAG:-s1l1} bash scripts/gpu_s1_qmm.sh
