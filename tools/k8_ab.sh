for pf in 0 2 3 4 2; do echo "pf $pf"; CCB_K8_PF=$pf timeout 300 python tools/k8_ab.py; done
