for f in "" "128,1" "160,1" "192,1" "256,1" "128,0" "0,4"; do
  echo "== force '$f'"; CCB_GEMM_FORCE=$f timeout 200 python tools/bench_gemm.py 802 2>&1 | tail -4 | cut -c1-125
done
