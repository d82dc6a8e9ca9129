timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "gather" 2>&1 | tail -3
timeout 300 python tools/k1_ab.py 2>&1 | tail -8
timeout 300 python tools/k1_ab.py 64 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -x -q -k "fullsize or prefill or tiers or replay" 2>&1 | tail -2
