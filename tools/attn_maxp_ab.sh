for v in p4 p8 p16 p4 p8 p16; do cp paper_2502_15734_b200/_lib_alt/$v.so paper_2502_15734_b200/_lib/libcc_b200.so; for r in 0.0 0.05 0.15; do echo "$v r=$r $(timeout 300 python tools/graph_step.py $r 2>&1 | grep graph)"; done; done
cp paper_2502_15734_b200/_lib_alt/p16.so paper_2502_15734_b200/_lib/libcc_b200.so
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "attention" 2>&1 | tail -1
