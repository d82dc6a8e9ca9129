for c in 8 16 24 32 12; do
  CCB_LOGITS_CTAS=$c timeout 300 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none -k regex:logits --csv --log-file gpurun_out/lg.csv python tools/profile_step.py > /dev/null 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/lg.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
print('ctas/sm $c logits us', [round(float(r[vi].replace(',',''))/1e3,1) for r in rows[1:]])
PY
done
