"""One config-2 attention launch (after warm-up) for ncu:
ncu --set full -k regex:attn -s 3 -c 1 python tools/attn_one.py [variant] [case]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import attn_ab  # noqa: E402,F401  (only for make/run; its main loop is guarded below)
from attn_ab import CASES, lib, make, run  # noqa: E402

variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
case = sys.argv[2] if len(sys.argv) > 2 else "config2 r=.15"
n_q, n, Hq, Hkv = CASES[case]
args = make(n_q, n, Hq, Hkv)
ctx = torch.empty((n_q, Hq * 128), dtype=torch.bfloat16, device="cuda")
lse = torch.empty((n_q, Hq), dtype=torch.float32, device="cuda")
lib.cc_debug_attn_variant(variant)
for _ in range(4):
    run(args, ctx, lse)
torch.cuda.synchronize()
