timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_kernels.py -x -q -k "decode or logits or gemv or argmax" 2>&1 | tail -2
run() {
  env "$@" timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_x.json 2> gpurun_out/dec_x.err
  python -c "
import json
d=json.loads(open('gpurun_out/dec_x.json').read().strip().splitlines()[-1])['decode']
print('$*', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
" || tail -3 gpurun_out/dec_x.err
}
run CCB_LOGITS_STREAM=0
run CCB_LOGITS_STREAM=1
