# decode ms/token: streaming GEMV only for the large projections (CCB_GS_MIN
# elements), per configuration, PDL on / off
run() {
  env "$@" timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_x.json 2> gpurun_out/dec_x.err
  python -c "
import json
d=json.loads(open('gpurun_out/dec_x.json').read().strip().splitlines()[-1])['decode']
print('$*', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
" || tail -3 gpurun_out/dec_x.err
}
run CCB_GEMV_STREAM=0 CCB_DECODE_PDL=0
run CCB_GEMV_STREAM=0 CCB_DECODE_PDL=1
run CCB_GEMV_STREAM=0 CCB_DECODE_PDL=1 CCB_DECODE_FUSED=1
for c in 0 3; do
  for m in 0 30000000 100000000; do
    run CCB_GS_CFG=$c CCB_GS_MIN=$m CCB_DECODE_PDL=0
    run CCB_GS_CFG=$c CCB_GS_MIN=$m CCB_DECODE_PDL=1
  done
done
