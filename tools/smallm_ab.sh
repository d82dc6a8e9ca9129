for M in 290 545; do
for m in auto "0,4" "256,0" "128,1" "208,2"; do
  if [ "$m" = auto ]; then env CCB_SW_DEBUG=1 timeout 100 python tools/bench_gemm.py $M 2>&1 | cut -c1-150 | sed "s/^/[$m] /";
  else CCB_GEMM_FORCE=$m timeout 100 python tools/bench_gemm.py $M 2>&1 | cut -c1-75 | sed "s/^/[$m] /"; fi
done; done
