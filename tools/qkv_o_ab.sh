for m in auto 160,0 192,0 224,0 256,0 208,2 176,2 0,4 160,1; do
  if [ "$m" = auto ]; then r=$(timeout 100 python tools/bench_gemm.py 802 2>&1 | grep -E "qkv|  o " | cut -c1-60 | tr '\n' ' ');
  else r=$(CCB_GEMM_FORCE=$m timeout 100 python tools/bench_gemm.py 802 2>&1 | grep -E "qkv|  o " | cut -c1-60 | tr '\n' ' '); fi
  echo "[$m] $r"
done
