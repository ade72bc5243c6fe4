# Round-2 session-3 evidence on the interleaved-chunk (R17) tree: gpu_evidence.sh (tests, smoke,
# default bench, reference arm, launch list, ncu --set full of the bench's decode launch), then
# the same config in the other chunk layouts and codecs, and the per-rank shares of §15.
TAG=${TAG:-s2ev} bash scripts/gpu_evidence.sh
OUT=gpurun_out/${TAG:-s2ev}
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['config']['chunk_symbols'], d['config'].get('chunk_mode'), round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d.get('fp8_out',{}).get('value',0),1), 'bits', round(d['bits_per_param'],4), d['clocks']['reasons'])" $1 $2; }
for mode in layer row; do
  timeout 900 python bench.py --chunk-mode $mode --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats > $OUT/bench_$mode.json 2> $OUT/bench_$mode.err
  line $OUT/bench_$mode.json "pair $mode"
done
for codec in word byte; do
  timeout 900 python bench.py --codec $codec --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats > $OUT/bench_$codec.json 2> $OUT/bench_$codec.err
  line $OUT/bench_$codec.json "$codec"
done
for G in 2 4 8; do
  for cs in 0 2048; do
    timeout 600 python bench.py --as-rank 0/$G --chunk-symbols $cs --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/share_G${G}_cs${cs}.json 2> $OUT/share_G${G}_cs${cs}.err
    line $OUT/share_G${G}_cs${cs}.json "share G=$G"
  done
done
