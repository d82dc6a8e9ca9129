"""Run one GEMM shape a few times (for ncu): python tools/gemm_one.py M N K epi [reps]
epi: store|resid|swiglu"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_15734_b200 import _native as N

M, Nn, K = (int(x) for x in sys.argv[1:4])
epi = {"store": N.EPI_STORE, "resid": N.EPI_RESID_ADD, "swiglu": N.EPI_SWIGLU, "gelu": N.EPI_GELU}[sys.argv[4]]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
A = torch.randn((M, K), device="cuda").bfloat16()
B = (torch.randn((Nn, K), device="cuda") / 64).bfloat16()
if epi == N.EPI_RESID_ADD:
    C = torch.zeros((M, Nn), device="cuda")
elif epi == N.EPI_SWIGLU:
    C = torch.empty((M, Nn // 2), device="cuda", dtype=torch.bfloat16)
else:
    C = torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    N.call("cc_gemm", N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, epi, N.BF16, 1, N.stream_ptr())
torch.cuda.synchronize()
