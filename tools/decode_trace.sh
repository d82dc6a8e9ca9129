timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -1
run() {
  env "$@" timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_x.json 2> gpurun_out/dec_x.err
  python -c "
import json
d=json.loads(open('gpurun_out/dec_x.json').read().strip().splitlines()[-1])['decode']
print('$*', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
" || tail -3 gpurun_out/dec_x.err
}
for t in 1 2; do run RUN=$t; done
echo "=== trace"; timeout 600 python tools/decode_trace.py 1 2>&1 | tail -3
