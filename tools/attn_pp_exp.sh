# ping-pong attention timing experiments + ncu source-level capture of variant 4 (config-2 full recompute)
timeout 300 python tools/attn_ab.py 4,4x16,4x32,4x64,4x128,4x192 30 "full,r=.15" 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_pp -s 3 -c 1 -o gpurun_out/pp_full python tools/attn_one.py 4 "config2 full" > gpurun_out/pp_ncu.log 2>&1; tail -3 gpurun_out/pp_ncu.log
