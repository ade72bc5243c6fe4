# A/B: DRAM bytes of one decode launch per variant (32 blocks) -> gpurun_out/dram_<so>.csv
set -x
for so in ${VARIANTS}; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_decode -s 1 -c 2 --csv --log-file gpurun_out/dram_$so.csv python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu --lam 230.2 > /dev/null 2>&1
done
