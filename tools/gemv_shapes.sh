for c in 0 3; do echo "== cfg $c"; CCB_GS_CFG=$c timeout 300 python tools/gemv_shapes.py; done
