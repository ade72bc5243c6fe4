# The adopted chunk / tail-block rule with bench defaults: shares, configs 2 / 3 / 5 (config 2 with
# its CPU-baseline parity leg over the mixed chunk lengths), and the reference arm on config 2.
OUT=gpurun_out/${TAG:-s2tail3}; mkdir -p $OUT
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['config']['chunk_symbols'], d['config'].get('tail_blocks_2048'), round(d['value'],1), round(d['roofline']['frac'],4), 'coded/nH', round((d.get('rate') or {}).get('coded_over_nH', 0),4), 'parity', (d.get('parity') or {}).get('mismatches'), d['clocks']['reasons'])" "$1" "$2"; }
for G in 2 4 8; do
  timeout 600 python bench.py --as-rank 0/$G --steps 20 --warmup 3 --no-e2e --no-cpu --lam 230.2 > $OUT/share_G$G.json 2> $OUT/share_G$G.err; line $OUT/share_G$G.json share_G$G
done
timeout 900 python bench.py --model llama-3.2-1b --steps 20 --warmup 3 --no-e2e > $OUT/config2.json 2> $OUT/config2.err; line $OUT/config2.json config2
timeout 1500 python bench.py --model llama-3-70b --blocks 10 --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/config5.json 2> $OUT/config5.err; line $OUT/config5.json config5
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > $OUT/config3.json 2> $OUT/config3.err; line $OUT/config3.json config3
timeout 600 python bench.py --impl reference --model llama-3.2-1b --steps 2 --warmup 1 > $OUT/ref_c2.json 2> $OUT/ref_c2.err; echo ref=$?; tail -c 400 $OUT/ref_c2.json
