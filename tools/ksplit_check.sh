timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "k_split or cta_pair or gemm" 2>&1 | tail -3
CCB_SW_DEBUG=1 timeout 300 python tools/bench_gemm.py 96 290 545 802 2>&1 | grep -v "^\[gemm_pair\]" | tail -16
CCB_PAIR_KSPLIT=0 timeout 300 python tools/bench_gemm.py 96 290 545 2>&1 | tail -12
CCB_SW_DEBUG=1 timeout 300 python tools/bench_gemm.py 290 2>&1 | grep "^\[gemm_pair\]" | sort | uniq | head
for k in 1 0; do CCB_PAIR_KSPLIT=$k timeout 900 python bench.py --tiers 0 --no-baselines --sweep --decode-steps 0 --no-cpu > gpurun_out/ks_$k.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/ks_$k.json').read().strip().splitlines()[-1])
print('ksplit=$k', d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d.get('recompute_sweep', {}).items()})"; done
