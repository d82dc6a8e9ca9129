for r in 0.0 0.05 0.10 0.15; do for k in 0 1; do echo "r=$r ksplit=$k $(CCB_PAIR_KSPLIT=$k timeout 300 python tools/graph_step.py $r 2>&1 | grep graph)"; done; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ks_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/ks_pytest.log
