for M in 290 545; do
echo "== default"; timeout 120 python tools/bench_gemm.py $M 2>&1 | tail -4 | cut -c1-120
echo "== pair (CCB_GEMM_FORCE=0,4)"; CCB_GEMM_FORCE=0,4 timeout 120 python tools/bench_gemm.py $M 2>&1 | tail -4 | cut -c1-120
echo "== dp bn256 (256,0)"; CCB_GEMM_FORCE=256,0 timeout 120 python tools/bench_gemm.py $M 2>&1 | tail -4 | cut -c1-120
done
