for v in 1 0 1; do
  CCB_RMSNORM_WARP=$v timeout 300 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none -k regex:"rmsnorm" --csv --log-file gpurun_out/rms.csv python tools/profile_step.py > /dev/null 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/rms.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value'); ki=h.index('Kernel Name')
ts=[float(r[vi].replace(',','')) for r in rows[1:]]
print('rmsnorm warp=$v', rows[1][ki][:24], 'avg us', round(sum(ts)/len(ts)/1e3,2), len(ts))
PY
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --tiers 0 --decode-steps 0 > gpurun_out/q_main.json 2> gpurun_out/q_main.err; python -c "
import json;d=json.loads(open('gpurun_out/q_main.json').read().strip().splitlines()[-1])
print('main', d['value'], d['ms_per_step'], d['e2e']['value'], d['ttft_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
timeout 900 python bench.py --config 70b --steps 3 --tiers 0 --decode-steps 0 > gpurun_out/q_70b.json 2> gpurun_out/q_70b.err; python -c "
import json;d=json.loads(open('gpurun_out/q_70b.json').read().strip().splitlines()[-1])
print('70b', d['value'], d['ms_per_step'], d['e2e']['value'], d['ttft_ms'])"
