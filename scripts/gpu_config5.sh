# config 5 per-rank share on one B200: 10 Llama-3-70B-shaped blocks (one of 8 ranks' shards):
# compress time (calibration + Alg. 1 for 10 blocks) and decode throughput of the shard
timeout 1500 python bench.py --model llama-3-70b --blocks 10 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/config5.json 2> gpurun_out/config5.err
echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/config5.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1), 'bits', round(d['bits_per_param'],4), 'encode_s', round(d['encode_s'],1), 'lambda', d['config']['lambda'])"
