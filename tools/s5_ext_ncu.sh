for e in 1 0; do CCB_ATTN_EXT=$e timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_pp" --csv --log-file gpurun_out/ext_$e.csv python tools/profile_step.py --ratio 0.0 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/ext_$e.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value'); ki=h.index('Kernel Name')
d=collections.defaultdict(list)
for r in rows[1:]: d[r[ki][:24]].append(float(r[vi].replace(',','')))
print('ext=$e', {k: (len(v), round(sum(v)/len(v)/1e3,2)) for k,v in d.items()})
PY
done
