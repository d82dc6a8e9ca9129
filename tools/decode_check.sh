timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 5 > gpurun_out/dec.json 2> gpurun_out/dec.err; echo "rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/dec.json').read().strip().splitlines()[-1])
print(json.dumps(d.get('decode')))
"
