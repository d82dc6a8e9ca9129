for r in 0.0 0.05; do for k in 0 1; do echo "r=$r ksplit=$k $(CCB_PAIR_KSPLIT=$k timeout 300 python tools/graph_step.py $r 2>&1 | grep graph)"; done; done
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r0m_launches.csv python tools/profile_step.py --ratio 0.0 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_summary.py launches gpurun_out/r0m_launches.csv > gpurun_out/r0m_launches.md 2>&1; head -16 gpurun_out/r0m_launches.md
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py -m gpu -x -q 2>&1 | tail -1
