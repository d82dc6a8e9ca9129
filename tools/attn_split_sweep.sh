timeout 600 python tools/attn_ab.py 4 20 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prefill.py -x -q -k "attention" 2>&1 | tail -1
timeout 900 python bench.py --config 70b --no-cpu > gpurun_out/r2f_70b_split.json 2> gpurun_out/r2f_70b_split.err; echo 70b rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/r2f_70b_split.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], [(k['kernel'], k.get('avg_launch_us'), k.get('frac')) for k in d.get('roofline_kernels', [])], d.get('clocks'))
"
