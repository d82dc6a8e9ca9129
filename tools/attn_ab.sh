# attention work-item split A/B at a given recompute ratio (default 0: question rows only, small grid)
R=${1:-0}
timeout 600 python -m pytest tests -m gpu -x -q -k "attention or prefill or fullsize or decode or segment" 2>&1 | tail -2
for v in "" "CCB_ATTN_NOSPLIT=1"; do
  echo "== ratio $R $v"
  env $v timeout 300 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/attn_v.csv python tools/profile_step.py --ratio $R > /dev/null 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/attn_v.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
ts=[float(r[vi].replace(',','')) for r in rows[1:] if 'attn_tc' in r[ki]]
tot=sum(float(r[vi].replace(',','')) for r in rows[1:] if r[h.index('Metric Name')]=='gpu__time_duration.sum')
print('attention launches', len(ts), 'avg us', round(sum(ts)/len(ts)/1e3,2) if ts else None, 'step total us', round(tot/1e3,1))
PY
done
