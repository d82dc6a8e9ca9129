timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "qkv_rope" 2>&1 | tail -2
timeout 300 python tools/qkv_rope_ab.py
