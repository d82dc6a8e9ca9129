timeout 600 python tools/profile_e2e.py 2>&1 | tail -45
timeout 300 python tools/bench_gemm.py 802 290 2>&1 | tail -12
