timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention_scattered" 2>&1 | tail -2
timeout 300 python tools/attn_ab.py 4,5,6 30 2>&1 | tail -5
