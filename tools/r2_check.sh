# GPU test suite + default bench line (round-2 status check); $1 = tag
T=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc=$? ; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?
python - <<PY
import json
d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'clocks', d.get('clocks'))
for k in d.get('roofline_kernels', []): print(k['kernel'], k.get('avg_launch_us'), k.get('frac'))
print('baselines', json.dumps(d.get('baselines'))[:600])
PY
