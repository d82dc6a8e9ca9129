nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2g_pytest.log
python __graft_entry__.py --smoke 2>&1 | tail -2
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/r2g_bench_$i.json 2> gpurun_out/r2g_bench_$i.err; echo bench$i rc=$?
  python - <<PY
import json
d=json.loads(open('gpurun_out/r2g_bench_$i.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'clocks', d.get('clocks'))
print('gemm', d['roofline']['frac'], [(k['kernel'], k.get('avg_launch_us'), k.get('frac')) for k in d.get('roofline_kernels', [])])
print('decode', d['decode']['ms_per_token'], d['decode']['roofline']['frac'])
print('miss', json.dumps(d['baselines'].get('miss_path_full_prefill'))[:200])
PY
done
timeout 900 python tools/profile_decode.py > /dev/null 2>&1
timeout 900 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2g_decode_launches.csv python tools/profile_decode.py > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_summary.py launches gpurun_out/r2g_decode_launches.csv > gpurun_out/r2g_decode_launches.md 2>&1; head -14 gpurun_out/r2g_decode_launches.md
timeout 600 python tools/decode_trace.py 2 > gpurun_out/r2g_decode_trace.txt 2>&1; tail -8 gpurun_out/r2g_decode_trace.txt
