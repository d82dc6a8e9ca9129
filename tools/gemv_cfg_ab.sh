# streaming-GEMV configurations (tools/bench_gemv.py per CCB_GS_CFG, plain and
# PDL-chained launches) vs the warp-per-row kernel, then decode ms/token
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for c in 0 1 2 3 4 5; do
  for pdl in 0 1; do echo "== cfg $c pdl $pdl"; CCB_BENCH_NOATTN=1 CCB_BENCH_PDL=$pdl CCB_GS_CFG=$c timeout 300 python tools/bench_gemv.py 2>&1 | grep gemv; done
done
for pdl in 0 1; do echo "== warp-per-row pdl $pdl"; CCB_BENCH_NOATTN=1 CCB_BENCH_PDL=$pdl CCB_GEMV_STREAM=0 timeout 300 python tools/bench_gemv.py 2>&1 | grep gemv; done
for c in 0 1 2 3 4 5; do
CCB_GS_CFG=$c timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_c$c.json 2> gpurun_out/dec_c$c.err
python -c "
import json
d=json.loads(open('gpurun_out/dec_c$c.json').read().strip().splitlines()[-1])['decode']
print('decode cfg $c', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
" || tail -5 gpurun_out/dec_c$c.err
done
CCB_DECODE_PDL=0 timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_nopdl.json 2> gpurun_out/dec_nopdl.err
python -c "
import json
d=json.loads(open('gpurun_out/dec_nopdl.json').read().strip().splitlines()[-1])['decode']
print('decode cfg 0 no pdl', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
"
