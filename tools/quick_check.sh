timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/q_main.json 2> gpurun_out/q_main.err; python -c "
import json;d=json.loads(open('gpurun_out/q_main.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['ttft_ms'], d['roofline']['frac'], d['kernel_time_share'], d['clocks']['sm_mhz'], d['decode']['ms_per_token'])"
timeout 900 python bench.py --config 70b --steps 3 > gpurun_out/q_70b.json 2> gpurun_out/q_70b.err; tail -c 600 gpurun_out/q_70b.json; tail -2 gpurun_out/q_70b.err
