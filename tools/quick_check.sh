timeout 900 python -m pytest tests -m gpu -x -q -k "decode or prefill or attention" 2>&1 | tail -2
timeout 600 python bench.py --tiers 0 --no-baselines > gpurun_out/q_main.json 2> gpurun_out/q_main.err; python -c "
import json;d=json.loads(open('gpurun_out/q_main.json').read().strip().splitlines()[-1])
print('main', d['value'], d['ms_per_step'], d['e2e']['value'], 'decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'], d['decode']['first_tokens'])"
