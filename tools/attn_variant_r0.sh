for v in 4 0 1 2 3 4; do echo "variant=$v r=0 $(CCB_ATTN_VARIANT=$v timeout 300 python tools/graph_step.py 0.0 2>&1 | grep graph)"; done
for v in 4 1; do echo "variant=$v r=0.05 $(CCB_ATTN_VARIANT=$v timeout 300 python tools/graph_step.py 0.05 2>&1 | grep graph)"; done
