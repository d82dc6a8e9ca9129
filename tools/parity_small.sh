export CCB_PARITY_OUT=gpurun_out/r2_parity_small.jsonl
rm -f $CCB_PARITY_OUT
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_decode.py tests/test_gpu_parallel.py -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
cat $CCB_PARITY_OUT | grep bf16
