timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prefill.py tests/test_gpu_parity_fullsize.py tests/test_gpu_replay.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu --tiers 0 --decode-steps 0 > gpurun_out/k8_8b.json 2> gpurun_out/k8_8b.err; echo "8b rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/k8_8b.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], json.dumps(d['baselines'].get('miss_path_full_prefill')))
"
timeout 900 python bench.py --config zipf > gpurun_out/k8_zipf.json 2> gpurun_out/k8_zipf.err; echo "zipf rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/k8_zipf.json').read().strip().splitlines()[-1])
print(d['value'], json.dumps(d.get('policies',{}).get('cachecraft')))
"
