# Round-2 session-2 A/B: pair-decoder variants (narrow 2·id LUT entries, restructured group
# loop), per-rank shares at chunk lengths that give whole rounds, and one ncu capture of k_search.
OUT=gpurun_out/${TAG:-s1ab}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "search or calib or config1 or sampled_rows" > $OUT/search_tests.log 2>&1; echo search_tests=$?; tail -3 $OUT/search_tests.log
python scripts/search_once.py > $OUT/search_time.log 2>&1; cat $OUT/search_time.log
VARIANTS="${VARIANTS:-ab_base.so ab_n.so ab_l.so ab_nl.so}" NCU=1 TAG=${TAG:-s1ab} bash scripts/gpu_ab_r2.sh
for spec in ${SHARES:-0/8:4608 0/8:2304 0/4:4608 0/4:3072 0/2:4608 0/2:3712 0/1:4608}; do
  r=${spec%%:*}; cs=${spec##*:}; tag=$(echo $r | tr / _)_$cs
  timeout 600 python bench.py --as-rank $r --chunk-symbols $cs --steps 20 --warmup 3 --no-e2e --no-cpu --no-stats --lam 230.2 > $OUT/share_$tag.json 2> $OUT/share_$tag.err
  python -c "import json; d=json.loads(open('$OUT/share_$tag.json').read().strip().splitlines()[-1]); s=d.get('per_rank_share') or {}; print('share $r cs=$cs', round(d['value'],1), 'GB/s frac', round(d['roofline']['frac'],4), 'bits', round(d['bits_per_param'],4), 'rounds', round(s.get('rounds',0),3), 'ms', round(d['ms_per_step'],4), d['clocks']['reasons'])"
done
if [ -z "$NOSEARCH" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_search -c 1 -o $OUT/search \
    python scripts/search_once.py > $OUT/search_ncu.log 2>&1; echo ncu_search=$?
python scripts/ncu_summary.py $OUT/search.ncu-rep > $OUT/search_summary.json 2>&1
fi
