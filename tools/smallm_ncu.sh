# what ncu says about the M = 290 pair GEMMs
timeout 300 ncu --set full --clock-control none -k regex:gemm -s 1 -c 1 -o gpurun_out/sm_qkv python tools/gemm_one.py 290 6144 4096 store 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:gemm -s 1 -c 1 -o gpurun_out/sm_down python tools/gemm_one.py 290 4096 14336 resid 3 > /dev/null 2>&1
for f in sm_qkv sm_down; do python tools/ncu_summary.py report gpurun_out/$f.ncu-rep $f 2>&1 | head -24; done
