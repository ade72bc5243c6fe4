# Chunk length A/B for partial-round shares (bench.choose_chunk): same build, same box.
OUT=gpurun_out/${TAG:-s2cab}; mkdir -p $OUT
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['config']['chunk_symbols'], round(d['value'],1), round(d['roofline']['frac'],4), 'rounds', round((d.get('per_rank_share') or {}).get('rounds', 0),3), 'bits', round(d['bits_per_param'],4))" "$1" "$2"; }
for G in 2 4 8; do for cs in 4096 4608; do
  timeout 600 python bench.py --as-rank 0/$G --chunk-symbols $cs --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --no-fp8 --lam 230.2 > $OUT/G${G}_$cs.json 2> $OUT/G${G}_$cs.err
  line $OUT/G${G}_$cs.json "G=$G"
done; done
for cs in 4096 4608 5632; do
  timeout 900 python bench.py --model llama-3.2-1b --chunk-symbols $cs --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --no-fp8 > $OUT/c2_$cs.json 2> $OUT/c2_$cs.err
  line $OUT/c2_$cs.json "config2"
done
for cs in 4096 4608; do
  timeout 900 python bench.py --model llama-3-70b --blocks 10 --chunk-symbols $cs --steps 10 --warmup 3 --no-e2e --no-cpu --no-stats --no-fp8 > $OUT/c5_$cs.json 2> $OUT/c5_$cs.err
  line $OUT/c5_$cs.json "config5"
done
