for r in 0.0 0.05 0.10; do for k in 0 1; do echo "ksplit=$k"; CCB_PAIR_KSPLIT=$k timeout 300 python tools/graph_step.py $r 2>&1 | grep "graph"; done; done
CCB_PAIR_KSPLIT=1 CCB_SW_DEBUG=1 timeout 300 python tools/graph_step.py 0.0 2>&1 | grep "gemm_pair" | sort | uniq
CCB_PAIR_KSPLIT=1 CCB_SW_DEBUG=1 timeout 300 python tools/graph_step.py 0.10 2>&1 | grep "gemm_pair" | sort | uniq
