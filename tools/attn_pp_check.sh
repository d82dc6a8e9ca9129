# ping-pong attention (variants 4/5): parity tests + A/B against the current variants + per-CTA trace
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention_scattered" 2>&1 | tail -3
timeout 600 python tools/attn_ab.py ${1:-0,1,4,5} 30 2>&1 | tail -12
timeout 300 python tools/attn_pp_trace.py r=.15 ${2:-5} 2>&1 | tail -20
timeout 300 python tools/attn_pp_trace.py full ${2:-5} 2>&1 | tail -8
