# config 2: Llama-3.2-1B-shaped layer set (16 blocks) — full quantise + encode (with λ
# calibration) and decode on one B200; the same bench contract, model switched
timeout 900 python bench.py --model llama-3.2-1b --steps 20 --warmup 3 --no-e2e > gpurun_out/config2.json 2> gpurun_out/config2.err
echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/config2.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['frac'],3), 'fp8', round(d['fp8_out']['value'],1), 'bits', round(d['bits_per_param'],4), 'encode_s', round(d['encode_s'],1), 'cpu', d['cpu_baseline']['value'])"
