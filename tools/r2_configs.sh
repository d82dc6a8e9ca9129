# round-2 numbers for every BASELINE config (N=1) with the committed kernels
for c in "8b --sweep" "8b-32k" "70b" "zipf"; do
  tag=$(echo $c | tr ' -' '__')
  timeout 1200 python bench.py --config $c > gpurun_out/r2cfg_${tag}.json 2> gpurun_out/r2cfg_${tag}.err; echo "$c rc=$?"
  python - <<PY
import json
d=json.loads(open('gpurun_out/r2cfg_${tag}.json').read().strip().splitlines()[-1])
print('  value', d.get('value'), 'ms', d.get('ms_per_step'), 'e2e', (d.get('e2e') or {}).get('value'), 'ttft', d.get('ttft_ms'))
print('  sweep', json.dumps(d.get('sweep'))[:500])
print('  roof', [(k['kernel'], k.get('avg_launch_us'), k.get('frac')) for k in d.get('roofline_kernels', [])], d.get('roofline', {}).get('frac'))
PY
done
timeout 900 python bench.py --impl reference > gpurun_out/r2cfg_reference.json 2> gpurun_out/r2cfg_reference.err; echo "reference rc=$?"; tail -c 600 gpurun_out/r2cfg_reference.json
