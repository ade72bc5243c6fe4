# R18 (grouped escapes) on one B200: its GPU tests, then the bench in R15 vs R18 (both with
# interleaved chunks, R17), and an ncu metric pass of each decode launch.
OUT=gpurun_out/${TAG:-s2r18}
mkdir -p $OUT
M=sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio
timeout 1500 python -m pytest tests/test_gpu_pair_codec.py tests/test_gpu_interleaved.py tests/test_gpu_parity.py "tests/test_gpu_fullsize.py::test_config3_every_symbol_matches_oracle_decode[pairg-il]" "tests/test_gpu_fullsize.py::test_config3_lossless_and_rate_properties[pairg-il]" -q -x > $OUT/tests.log 2>&1; echo tests=$?; tail -2 $OUT/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?; tail -1 $OUT/smoke.log
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['config']['chunk_symbols'], d['config'].get('chunk_mode'), round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d.get('fp8_out',{}).get('value',0),1), 'bits', round(d['bits_per_param'],4), d['clocks']['reasons'])" $1 $2; }
for rep in 1 2; do
for codec in pair pairg; do
  timeout 900 python bench.py --codec $codec --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/bench_${codec}_$rep.json 2> $OUT/bench_${codec}_$rep.err
  line $OUT/bench_${codec}_$rep.json "$codec"
done
done
for codec in pair pairg; do
  ncu --metrics $M --clock-control none -k regex:k_decode_p -c 2 --csv \
     python bench.py --codec $codec --profile --steps 1 --warmup 1 --no-e2e --no-cpu --lam 230.2 > $OUT/ncu_$codec.csv 2> $OUT/ncu_$codec.err
  echo ncu_$codec=$?
done
for codec in pair pairg; do echo $codec; python scripts/ncu_csv_summary.py $OUT/ncu_$codec.csv 2>&1 | tail -3; done
if [ -n "$FULL" ]; then
  ncu --set full --clock-control none --import-source on -k regex:k_decode -s 1 -c 2 -o $OUT/decode \
      python bench.py --codec pairg --profile --steps 1 --warmup 1 --no-e2e --no-cpu --lam 230.2 > $OUT/full_bench.log 2>&1; echo full=$?
  python scripts/ncu_summary.py $OUT/decode.ncu-rep > $OUT/summary.json 2>&1
  python -c "
import json; d=json.load(open('$OUT/summary.json'))
for x in d: print(x['kernel'], x.get('gpu__time_duration.sum'), x.get('smsp__issue_active.avg.pct_of_peak_sustained_active'), x.get('stalls_per_issue'))
"
  ncu -i $OUT/decode.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[2:4]:
    for k,v in zip(h,r):
        if ('l1tex__data_pipe' in k or 'l1tex__lsu' in k or 'lsuin_requests' in k or 'pipe_lsu' in k) and v not in ('','0'): print(k, v)
    print('--')
" | head -60
fi
