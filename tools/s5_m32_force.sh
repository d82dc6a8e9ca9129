echo "default $(timeout 300 python tools/graph_step.py 0.0 2>&1 | grep graph)"
for f in "0,4" "2,5" "3,5" "4,5" "6,5"; do echo "force=$f $(CCB_GEMM_FORCE=$f timeout 300 python tools/graph_step.py 0.0 2>&1 | grep graph)"; done
echo "default $(timeout 300 python tools/graph_step.py 0.0 2>&1 | grep graph)"
