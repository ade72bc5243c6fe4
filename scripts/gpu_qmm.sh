# config 4 (fused decode -> tcgen05 GEMM): timings at chunk 2048 / 1024 and one ncu --set full capture
set -x
OUT=gpurun_out/${TAG:-qmm}
mkdir -p $OUT
for cs in ${CS_LIST:-2048 1024}; do
  timeout 300 python scripts/bench_qmatmul.py --cs $cs --codec ${CODEC:-word} > $OUT/bench_cs$cs.json 2> $OUT/bench_cs$cs.err; echo bench$cs=$?
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qmatmul -c 2 -o $OUT/qmm \
      python scripts/bench_qmatmul.py --cs ${NCU_CS:-2048} --codec ${CODEC:-word} --profile > $OUT/ncu.log 2>&1; echo ncu=$?
  python scripts/ncu_summary.py $OUT/qmm.ncu-rep > $OUT/summary.json 2>&1
fi
