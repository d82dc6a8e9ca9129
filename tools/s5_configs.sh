timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "concurrent_streams or k_split" 2>&1 | tail -1
for c in 8b-32k 70b zipf; do timeout 1500 python bench.py --config $c > gpurun_out/s5c_$c.json 2> gpurun_out/s5c_$c.err; echo "$c rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/s5c_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d.get('ms_per_step'), 'e2e', d.get('e2e',{}).get('value'), 'ttft', d.get('ttft_ms'), 'roof', d['roofline']['kernel'], d['roofline']['frac'], [(k['kernel'], k.get('frac')) for k in d.get('roofline_kernels', [])], {k: v for k, v in d.get('baselines', {}).items() if 'speedup' in k})" 2>&1 | tail -2; done
