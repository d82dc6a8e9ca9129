timeout 400 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_attn" --csv --log-file gpurun_out/da.csv python tools/profile_decode.py > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/da.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value'); ki=h.index('Kernel Name')
d=collections.defaultdict(list)
for r in rows[1:]: d[r[ki][:30]].append(float(r[vi].replace(',','')))
print({k: round(sum(v)/len(v)/1e3,2) for k,v in d.items()})
PY
timeout 900 python -m pytest tests -m gpu -x -q -k "decode" 2>&1 | tail -1
timeout 600 python bench.py --tiers 0 --no-baselines > gpurun_out/q_main.json 2> gpurun_out/q_main.err; python -c "
import json;d=json.loads(open('gpurun_out/q_main.json').read().strip().splitlines()[-1])
print('main', d['value'], 'decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'], d['decode']['first_tokens'])"
