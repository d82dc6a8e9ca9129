timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -k "qkv_matches" 2>&1 | grep -E "Error|error|passed|failed" | head -10
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_decode.py -x -q -k "qkv_matches and 300" 2>&1 | grep -v "^    \|^=========     Host\|^$" | head -40
