for c in 8b-32k 70b; do
timeout 1500 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tr_$c.csv python tools/profile_step.py --config $c > gpurun_out/tr_$c.log 2>&1; echo "$c ncu rc=$?"; tail -2 gpurun_out/tr_$c.log
python tools/traffic_json.py gpurun_out/tr_$c.csv > gpurun_out/traffic_$c.json; cat gpurun_out/traffic_$c.json | head -22
python tools/ncu_summary.py launches gpurun_out/tr_$c.csv > gpurun_out/tr_$c.md 2>&1; head -16 gpurun_out/tr_$c.md
done
