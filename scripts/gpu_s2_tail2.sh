# Rank shares with the last k blocks in 2048-symbol chunks (4096 elsewhere) vs the 4608 rule.
OUT=gpurun_out/${TAG:-s2tail2}; mkdir -p $OUT
run() {  # label args...
  local tag=$1; shift
  timeout 900 python bench.py "$@" --steps 20 --warmup 3 --no-cpu --no-e2e > $OUT/$tag.json 2> $OUT/$tag.err
  python -c "import json; d=json.loads(open('$OUT/$tag.json').read().strip().splitlines()[-1]); print('$tag', d['config']['chunk_symbols'], round(d['value'],1), round(d['roofline']['frac'],4), 'coded/nH', round(d['rate']['coded_over_nH'],4), 'max', round(d['rate']['coded_over_nH_max_block'],4))"
}
run G2_k0 --as-rank 0/2 --lam 230.2 --chunk-symbols 4096
run G2_k2 --as-rank 0/2 --lam 230.2 --chunk-symbols 4096 --tail-blocks 2
run G4_4608 --as-rank 0/4 --lam 230.2 --chunk-symbols 4608
run G4_k1 --as-rank 0/4 --lam 230.2 --chunk-symbols 4096 --tail-blocks 1
run G8_4608 --as-rank 0/8 --lam 230.2 --chunk-symbols 4608
run G8_k1 --as-rank 0/8 --lam 230.2 --chunk-symbols 4096 --tail-blocks 1
run c5_k0 --model llama-3-70b --blocks 10 --chunk-symbols 4096
run c5_k1 --model llama-3-70b --blocks 10 --chunk-symbols 4096 --tail-blocks 1
run c2_k3 --model llama-3.2-1b --chunk-symbols 4096 --tail-blocks 3
run c2_k4 --model llama-3.2-1b --chunk-symbols 4096 --tail-blocks 4
run c2_k5 --model llama-3.2-1b --chunk-symbols 4096 --tail-blocks 5
