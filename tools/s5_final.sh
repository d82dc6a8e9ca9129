nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
python __graft_entry__.py --smoke 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/s5f_bench.json 2> gpurun_out/s5f_bench.err; echo bench rc=$?
timeout 900 python bench.py --sweep --no-baselines --tiers 0 --decode-steps 0 --no-cpu > gpurun_out/s5f_sweep.json 2> gpurun_out/s5f_sweep.err; echo sweep rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5f_ref.json 2> gpurun_out/s5f_ref.err; echo ref rc=$?
python - <<PY
import json
d=json.loads(open('gpurun_out/s5f_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'ttft', d.get('ttft_ms'), 'clocks', d.get('clocks'))
print(json.dumps(d['roofline']))
for k in d.get('roofline_kernels', []): print(k['kernel'], k.get('avg_launch_us'), k.get('frac'), k.get('traffic'))
print('decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'])
b=d['baselines']; print('full', b['full_recompute_ours']['ms_per_step'], 'cublas', b.get('full_recompute_cublas_cudnn_sdpa'), 'ttft', json.dumps(b.get('public_api_ttft')))
print('miss', json.dumps(b.get('miss_path_full_prefill'))[:300])
s=json.loads(open('gpurun_out/s5f_sweep.json').read().strip().splitlines()[-1]); print('sweep', s['value'], {k: (v['ms'], round(v['tokens_per_s'])) for k, v in s.get('recompute_sweep', {}).items()})
r=json.loads(open('gpurun_out/s5f_ref.json').read().strip().splitlines()[-1]); print('ref', r.get('value'), r.get('unit'), r.get('cpu_baseline'))
PY
