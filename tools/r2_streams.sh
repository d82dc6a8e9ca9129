for k in 4 6 10; do
  timeout 900 python bench.py --streams $k --no-baselines --no-cpu --tiers 0 --decode-steps 0 > gpurun_out/r2st_$k.json 2> gpurun_out/r2st_$k.err
  python -c "
import json
d=json.loads(open('gpurun_out/r2st_$k.json').read().strip().splitlines()[-1])
print('streams $k', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'single', d['single_request']['value'])
"
done
