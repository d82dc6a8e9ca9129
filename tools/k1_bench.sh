timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "gather" 2>&1 | tail -1
timeout 300 python tools/k1_ab.py 2>&1 | tail -6
timeout 300 python tools/k1_ab.py 64 2>&1 | tail -6
for m in 0 1; do CCB_K1_LDG=$m timeout 900 python bench.py --tiers 0 --no-baselines > gpurun_out/k1b_$m.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/k1b_$m.json').read().strip().splitlines()[-1])
print('ldg=$m', d['value'], d['ms_per_step'], [(k['kernel'], k.get('avg_launch_us'), k.get('frac')) for k in d.get('roofline_kernels', [])][:1], d['clocks']['sm_mhz'])"; done
