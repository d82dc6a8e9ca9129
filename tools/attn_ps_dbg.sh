timeout 300 python tools/attn_ab.py 6,6x1,6x2,6x3,4 20 "r=.15,full" 2>&1 | tail -3
