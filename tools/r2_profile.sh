# config-2 step launch list with DRAM bytes (ncu, cold caches / serialised), the
# traffic json for bench.py, one --set full capture of the attention kernel
# (config 2 shape) and the default bench line.   $1 = tag
T=${1:-r2}
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_step.py > /dev/null 2>&1; echo ncu-list rc=$?
python tools/traffic_json.py gpurun_out/${T}_launches.csv > gpurun_out/traffic_8b.json && cp gpurun_out/traffic_8b.json profiles/traffic_8b.json
python tools/ncu_summary.py launches gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.md 2>&1; head -40 gpurun_out/${T}_launches.md
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_pp -s 3 -c 1 -o gpurun_out/${T}_attn python tools/attn_one.py 4 "config2 r=.15" > /dev/null 2>&1; echo ncu-attn rc=$?
python tools/ncu_summary.py report gpurun_out/${T}_attn.ncu-rep "attention (ping-pong, config 2)" > gpurun_out/${T}_attn.md 2>&1; head -30 gpurun_out/${T}_attn.md
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?
python - <<PY
import json
d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'clocks', d.get('clocks'))
print(json.dumps(d['roofline']))
for k in d.get('roofline_kernels', []): print(k['kernel'], k.get('avg_launch_us'), k.get('frac'), k.get('traffic'))
PY
