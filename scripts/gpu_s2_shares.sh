# Per-rank shares (§8(e) split) and configs 2 / 5 with the chunk-length rule of bench.choose_chunk.
OUT=gpurun_out/${TAG:-s2sh}; mkdir -p $OUT
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['config']['codec'], d['config']['chunk_symbols'], d['config'].get('chunk_mode'), round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d.get('fp8_out',{}).get('value',0),1), 'bits', round(d['bits_per_param'],4), 'enc_s', round(d.get('encode_s',0),1), d['clocks']['reasons'])" "$1" "$2"; }
for G in 2 4 8; do
  timeout 600 python bench.py --as-rank 0/$G --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/share_G$G.json 2> $OUT/share_G$G.err
  line $OUT/share_G$G.json "share_G$G"
done
timeout 900 python bench.py --model llama-3.2-1b --steps 20 --warmup 3 --no-e2e --no-cpu > $OUT/config2.json 2> $OUT/config2.err
line $OUT/config2.json "config2"
timeout 900 python bench.py --model llama-3.2-1b --chunk-symbols 4096 --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats > $OUT/config2_4096.json 2> $OUT/config2_4096.err
line $OUT/config2_4096.json "config2_4096"
timeout 1500 python bench.py --model llama-3-70b --blocks 10 --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/config5.json 2> $OUT/config5.err
line $OUT/config5.json "config5"
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats > $OUT/config3.json 2> $OUT/config3.err
line $OUT/config3.json "config3"
