for p in 1 0 1; do
  CCB_PDL=$p timeout 300 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pdl_$p.csv python tools/profile_step.py > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/pdl_$p.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
tot=collections.defaultdict(float)
for r in rows[1:]: tot[r[ki].split('(')[0][-28:]]+=float(r[vi].replace(',',''))
print('PDL=$p total', round(sum(tot.values())/1e3,1), {k: round(v/1e3,0) for k,v in sorted(tot.items(), key=lambda x:-x[1])[:7]})
PY
done
CCB_PDL=1 timeout 300 python tools/step_time.py 2>&1 | tail -6
