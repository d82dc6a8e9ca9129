#!/bin/bash
# time each GEMM shape at M=802 under forced (BN, splits)
for f in 256,1 256,2 256,3 256,5 128,1 128,2; do
  echo "== CCB_GEMM_FORCE=$f"; CCB_GEMM_FORCE=$f timeout 120 python tools/bench_gemm.py 802 | cut -c1-75
done
