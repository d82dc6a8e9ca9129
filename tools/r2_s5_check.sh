nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s5_pytest.log
python __graft_entry__.py --smoke 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo bench rc=$?
python - <<PY
import json
d=json.loads(open('gpurun_out/s5_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'clocks', d.get('clocks'))
print('gemm', d['roofline']['frac'], [(k['kernel'], k.get('avg_launch_us'), k.get('frac')) for k in d.get('roofline_kernels', [])])
print('decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'])
PY
