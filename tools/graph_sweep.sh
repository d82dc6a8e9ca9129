for r in 0.0 0.05 0.10 0.15; do for k in 0 1; do echo "ksplit=$k"; CCB_PAIR_KSPLIT=$k timeout 300 python tools/graph_step.py $r 2>&1 | grep ms/step; done; done
