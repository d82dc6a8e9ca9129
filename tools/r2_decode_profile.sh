# Decode round-2 evidence: smoke, the decode launch list (ncu, cold caches /
# serialised), the in-kernel timeline, one --set full capture of the
# streaming GEMV (gate/up) and of the attention step.   $1 = tag
T=${1:-r2_decode}
python __graft_entry__.py --smoke 2>&1 | tail -3
timeout 900 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_decode.py > /dev/null 2>&1; echo ncu-list rc=$?
python tools/ncu_summary.py launches gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.md 2>&1; head -30 gpurun_out/${T}_launches.md
timeout 600 python tools/decode_trace.py 2 > gpurun_out/${T}_trace.txt 2>&1; tail -16 gpurun_out/${T}_trace.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_stream_kernel -s 100 -c 1 -o gpurun_out/${T}_gemv python tools/profile_decode.py > /dev/null 2>&1; echo ncu-gemv rc=$?
python tools/ncu_summary.py report gpurun_out/${T}_gemv.ncu-rep "decode streaming GEMV" > gpurun_out/${T}_gemv.md 2>&1; head -30 gpurun_out/${T}_gemv.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_tc -s 20 -c 1 -o gpurun_out/${T}_attn python tools/profile_decode.py > /dev/null 2>&1; echo ncu-attn rc=$?
python tools/ncu_summary.py report gpurun_out/${T}_attn.ncu-rep "decode attention step" > gpurun_out/${T}_attn.md 2>&1; head -30 gpurun_out/${T}_attn.md
