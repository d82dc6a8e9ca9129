# GPU test suite + default bench line (round-2 status check)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_pytest.log 2>&1; echo pytest rc=$? ; tail -5 gpurun_out/r2s3_pytest.log
timeout 600 python bench.py > gpurun_out/r2s3_bench.json 2> gpurun_out/r2s3_bench.err; echo bench rc=$?; tail -c 1500 gpurun_out/r2s3_bench.json
