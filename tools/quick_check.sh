timeout 300 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none -k regex:logits --csv --log-file gpurun_out/lg.csv python tools/profile_step.py > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/lg.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
print('logits us', [round(float(r[vi].replace(',',''))/1e3,1) for r in rows[1:]])
PY
timeout 900 python -m pytest tests -m gpu -x -q -k "logits or decode or prefill" 2>&1 | tail -1
timeout 600 python bench.py --tiers 0 --no-baselines > gpurun_out/q_main.json 2> gpurun_out/q_main.err; python -c "
import json;d=json.loads(open('gpurun_out/q_main.json').read().strip().splitlines()[-1])
print('main', d['value'], d['ms_per_step'], 'decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'], d['decode']['first_tokens'])"
