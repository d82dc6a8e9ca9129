timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention_scattered" 2>&1 | tail -2
timeout 300 python tools/attn_ab.py 0,1,4,5 20 2>&1 | tail -6
timeout 300 python tools/attn_ab.py 4@16/3,4@12/4,4@20/2,4@24/2 20 "r=.15" 2>&1 | tail -2
timeout 300 python tools/attn_pp_trace.py r=.15 4 2>&1 | grep -E "==|cycles|totals|busiest"
