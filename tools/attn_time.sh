timeout 300 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none -k regex:attn --csv --log-file gpurun_out/at.csv python tools/profile_step.py > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/at.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
ts=[float(r[vi].replace(',','')) for r in rows[1:]]
print('attention avg us', round(sum(ts)/len(ts)/1e3,2), len(ts))
PY
