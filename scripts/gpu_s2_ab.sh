# Session-3 A/B of R18 decoder variants (ab_*.so) with the bench's encoding (pairg, interleaved):
# VALS (bf16x2 value table) vs codes, and SKIP00; then the GPU parity tests of the default build.
OUT=gpurun_out/${TAG:-s2ab}
mkdir -p $OUT
VARIANTS="${VARIANTS:-ab_v1s0.so ab_v0s0.so ab_v1s1.so}" NCU=1 TAG=${TAG:-s2ab} BENCH_ARGS="--codec pairg" bash scripts/gpu_ab_r2.sh
for so in ${VARIANTS:-ab_v1s0.so ab_v0s0.so ab_v1s1.so}; do echo $so; python scripts/ncu_csv_summary.py $OUT/ncu_$so.csv 2>&1 | tail -2; done
timeout 1500 python -m pytest tests/test_gpu_pair_codec.py tests/test_gpu_interleaved.py tests/test_gpu_parity.py tests/test_gpu_qmatmul.py tests/test_gpu_rowchunk.py -q > $OUT/tests.log 2>&1; echo tests=$?; tail -3 $OUT/tests.log
