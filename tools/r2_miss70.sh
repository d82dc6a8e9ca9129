timeout 900 python bench.py > gpurun_out/r2m_8b.json 2> gpurun_out/r2m_8b.err; echo "8b rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r2m_8b.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], json.dumps(d['baselines'].get('miss_path_full_prefill')))
"
timeout 1500 python bench.py --config 70b > gpurun_out/r2m_70b.json 2> gpurun_out/r2m_70b.err; echo "70b rc=$?"; tail -3 gpurun_out/r2m_70b.err
python -c "
import json
d=json.loads(open('gpurun_out/r2m_70b.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('ttft_ms'), json.dumps(d.get('baselines'))[:700])
print([(k['kernel'], k.get('avg_launch_us'), k.get('frac')) for k in d.get('roofline_kernels', [])], d['roofline'].get('frac'))
"
