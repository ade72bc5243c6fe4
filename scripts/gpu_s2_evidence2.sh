# Round-2 evidence on the R18 tree (bench default: pair codec with grouped escapes R18 over
# interleaved chunks R17): gpu_evidence.sh (all GPU tests, smoke, bench, reference arm, launch
# list, ncu --set full), the other encodings on the same box, the per-rank shares of §8(e),
# configs 2 and 5, and the fused GEMM (config 4) with R15 vs R18 row-chunked streams.
TAG=${TAG:-s2ev2} bash scripts/gpu_evidence.sh
OUT=gpurun_out/${TAG:-s2ev2}
line() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['config']['codec'], d['config']['chunk_symbols'], d['config'].get('chunk_mode'), round(d['value'],1), round(d['roofline']['frac'],4), 'fp8', round(d.get('fp8_out',{}).get('value',0),1), 'bits', round(d['bits_per_param'],4), 'enc_s', round(d.get('encode_s',0),1), d['clocks']['reasons'])" "$1" "$2"; }
for spec in "pair interleaved" "pairg layer" "pairg row" "word layer" "byte layer"; do
  set -- $spec
  timeout 900 python bench.py --codec $1 --chunk-mode $2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats > $OUT/bench_$1_$2.json 2> $OUT/bench_$1_$2.err
  line $OUT/bench_$1_$2.json "enc"
done
for G in 2 4 8; do
  timeout 600 python bench.py --as-rank 0/$G --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/share_G$G.json 2> $OUT/share_G$G.err
  line $OUT/share_G$G.json "share_G$G"
done
timeout 900 python bench.py --model llama-3.2-1b --steps 20 --warmup 3 --no-e2e > $OUT/config2.json 2> $OUT/config2.err
line $OUT/config2.json "config2"
timeout 1500 python bench.py --model llama-3-70b --blocks 10 --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/config5.json 2> $OUT/config5.err
line $OUT/config5.json "config5"
for codec in pair pairg; do
  for cs in 4096 2048; do
    timeout 600 python scripts/bench_qmatmul.py --codec $codec --cs $cs > $OUT/qmm_${codec}_$cs.json 2> $OUT/qmm_${codec}_$cs.err
    python -c "import json; d=json.load(open('$OUT/qmm_${codec}_$cs.json')); print('qmm $codec cs=$cs', 'b1', round(d['batch1']['fused_group_ms'],4), round(d['batch1']['fused_group_decode_Tsym_per_s'],3), 'b64', round(d['batch64']['fused_group_ms'],4), round(d['batch64']['fused_group_decode_Tsym_per_s'],3), 'dense', round(d['batch1']['dense_bf16_cublas_ms'],4), 'dec+cublas', round(d['batch1']['decode_then_cublas_ms'],4), 'bits', round(d['effective_bits'],4))"
  done
done
