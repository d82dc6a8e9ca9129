for M in 64 160 290 545 802; do timeout 120 python tools/bench_gemm.py $M 2>&1 | tail -4 | cut -c1-120; done
timeout 900 python bench.py --sweep --no-baselines --no-cpu --tiers 0 --decode-steps 0 > gpurun_out/sw.json 2> gpurun_out/sw.err; echo "rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1])
print(d['value'], json.dumps(d.get('recompute_sweep')))
"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm" 2>&1 | tail -2
