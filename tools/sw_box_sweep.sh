#!/bin/bash
# unit-table swap GEMM: TMA box rows sweep at M=802 (forced table plan) vs auto
echo "== auto"; timeout 200 python tools/bench_gemm.py 802 | cut -c1-75
for b in 32 64 128 256; do
  echo "== table, box $b"; CCB_SW_DEBUG=1 CCB_SW_BOX=$b CCB_GEMM_FORCE=0,3 timeout 200 python tools/bench_gemm.py 802 2>&1 | cut -c1-110
done
