timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "attention" 2>&1 | tail -1
CCB_ATTN_EXT=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "attention" 2>&1 | tail -3
for r in 0.0 0.05 0.15; do for e in 0 -1 1; do if [ "$e" = "-1" ]; then unset CCB_ATTN_EXT; else export CCB_ATTN_EXT=$e; fi; echo "r=$r ext=$e $(timeout 300 python tools/graph_step.py $r 2>&1 | grep graph)"; done; done
