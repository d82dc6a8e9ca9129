timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5l_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/s5l_pytest.log
python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/s5l_bench.json 2> gpurun_out/s5l_bench.err; echo bench rc=$?
python - <<PY
import json
d=json.loads(open('gpurun_out/s5l_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'ttft', d.get('ttft_ms'), 'clocks', d.get('clocks'), 'launches', d.get('gpu_launches'), 'simt', d.get('bf16_simt_launches'))
print('gemm', d['roofline']['frac'], [(k['kernel'], k.get('avg_launch_us'), k.get('frac')) for k in d.get('roofline_kernels', [])], 'decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'])
PY
