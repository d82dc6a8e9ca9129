# Round-end measurement set (one box): GPU tests, default bench (+ sweep), configs 3/4/5,
# reference arm, launch list of the config-2 step with DRAM bytes.
set -x
timeout 1000 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/h_tests.log; cat gpurun_out/h_tests.log
timeout 900 python bench.py --sweep > gpurun_out/h_main.json 2> gpurun_out/h_main.err; tail -c 400 gpurun_out/h_main.json
timeout 600 python bench.py --config 8b-32k > gpurun_out/h_32k.json 2> gpurun_out/h_32k.err; tail -c 300 gpurun_out/h_32k.json
timeout 900 python bench.py --config 70b --steps 3 > gpurun_out/h_70b.json 2> gpurun_out/h_70b.err; tail -c 300 gpurun_out/h_70b.json
timeout 600 python bench.py --config zipf > gpurun_out/h_zipf.json 2> gpurun_out/h_zipf.err; tail -c 300 gpurun_out/h_zipf.json
timeout 600 python bench.py --impl reference > gpurun_out/h_ref.json 2> gpurun_out/h_ref.err; tail -c 300 gpurun_out/h_ref.json
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_h.csv python tools/profile_step.py > /dev/null 2>&1
ls -la gpurun_out/h_*.json gpurun_out/launches_h.csv
