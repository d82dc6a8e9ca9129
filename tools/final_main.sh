# Final config-2 measurement (bench with sweep) + launch list with DRAM bytes
timeout 900 python bench.py --sweep > gpurun_out/z_main.json 2> gpurun_out/z_main.err; tail -c 300 gpurun_out/z_main.json
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_z.csv python tools/profile_step.py > /dev/null 2>&1
ls -la gpurun_out/z_main.json gpurun_out/launches_z.csv
