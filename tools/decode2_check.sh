# Decode round-2 check: kernel tests, the GEMV micro-bench and decode ms/token
# under each switch (fused attention step, PDL, streaming GEMV).
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_gemv.py 2>&1 | tail -8
CCB_GEMV_STREAM=0 timeout 300 python tools/bench_gemv.py 2>&1 | tail -8
for v in "1 1 1" "1 0 1" "0 0 1" "1 1 0" "0 0 0"; do
set -- $v
CCB_DECODE_FUSED=$1 CCB_DECODE_PDL=$2 CCB_GEMV_STREAM=$3 timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_$1$2$3.json 2> gpurun_out/dec_$1$2$3.err
python -c "
import json
d=json.loads(open('gpurun_out/dec_$1$2$3.json').read().strip().splitlines()[-1])['decode']
print('fused/pdl/stream $1$2$3', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
" || tail -5 gpurun_out/dec_$1$2$3.err
done
