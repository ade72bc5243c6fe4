# Round-2 A/B of decoder variants (.so files under paper_2601_22787_b200/): parity tests of the
# pair codec, two short bench lines each (fixed λ, no e2e / cpu legs), then one ncu pass of the
# bf16 decode launch with instruction / issue / shared-memory counters.
# usage: VARIANTS="ab_base.so ab_b.so" TAG=x bash scripts/gpu_ab_r2.sh
OUT=gpurun_out/${TAG:-ab}
mkdir -p $OUT
M=sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio
for so in ${VARIANTS}; do
  EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python -m pytest tests/test_gpu_pair_codec.py -x -q > $OUT/test_$so.log 2>&1
  t=$?
  for rep in 1 2; do
    EQ_LIB=$PWD/paper_2601_22787_b200/$so timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --lam 230.2 ${BENCH_ARGS} > $OUT/bench_${so}_$rep.log 2>&1
    echo "$so rep$rep tests=$t $(python -c "import json,sys; d=json.loads(open('$OUT/bench_${so}_$rep.log').read().strip().splitlines()[-1]); print(round(d['value'],1), 'GB/s', round(d['roofline']['frac'],4), 'fp8', round(d.get('fp8_out',{}).get('value',0),1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])")"
  done
  if [ -n "$NCU" ]; then
    EQ_LIB=$PWD/paper_2601_22787_b200/$so ncu --metrics $M --clock-control none -k regex:k_decode -c 2 --csv \
      python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu --lam 230.2 ${BENCH_ARGS} > $OUT/ncu_$so.csv 2> $OUT/ncu_$so.err
  fi
done
