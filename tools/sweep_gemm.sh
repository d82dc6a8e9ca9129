#!/bin/bash
# time each GEMM shape under forced tilings (bn, mode: 0 data-parallel, 1 stream-K hybrid)
M=${1:-802}
echo "== auto"; timeout 120 python tools/bench_gemm.py $M | cut -c1-75
for f in 256,0 256,1 192,0 192,1 128,0 128,1; do
  echo "== CCB_GEMM_FORCE=$f"; CCB_GEMM_FORCE=$f timeout 120 python tools/bench_gemm.py $M | cut -c1-75
done
