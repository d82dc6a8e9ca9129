# session-5 evidence: GPU suite, step launch list + traffic json, --set full of
# the TMA-staged K1, default bench line.
T=s5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/${T}_pytest.log
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_step.py > /dev/null 2>&1; echo ncu-list rc=$?
python tools/traffic_json.py gpurun_out/${T}_launches.csv > gpurun_out/traffic_8b.json && cp gpurun_out/traffic_8b.json profiles/traffic_8b.json
python tools/ncu_summary.py launches gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.md 2>&1; head -30 gpurun_out/${T}_launches.md
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_rope_bulk -c 1 -o gpurun_out/${T}_k1 python tools/k1_ab.py > /dev/null 2>&1; echo ncu-k1 rc=$?
python tools/ncu_summary.py report gpurun_out/${T}_k1.ncu-rep "K1 TMA-staged gather+RoPE (config 2 shape)" > gpurun_out/${T}_k1.md 2>&1; head -40 gpurun_out/${T}_k1.md
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?
python - <<PY
import json
d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'clocks', d.get('clocks'))
print(json.dumps(d['roofline']))
for k in d.get('roofline_kernels', []): print(k['kernel'], k.get('avg_launch_us'), k.get('frac'), k.get('traffic'))
print('decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'])
PY
