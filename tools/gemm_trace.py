"""Per-CTA epilogue timeline of one GEMM (debug): python tools/gemm_trace.py M N K epi"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_15734_b200 import _native as N

M, Nn, K = (int(x) for x in sys.argv[1:4])
epi = {"store": N.EPI_STORE, "resid": N.EPI_RESID_ADD, "swiglu": N.EPI_SWIGLU}[sys.argv[4]]
A = torch.randn((M, K), device="cuda").bfloat16()
B = (torch.randn((Nn, K), device="cuda") / 64).bfloat16()
C = torch.zeros((M, Nn), device="cuda") if epi == N.EPI_RESID_ADD else torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)
tr = torch.zeros((148, 8, 8), dtype=torch.int64, device="cuda")
lib = N.lib()
run = lambda: N.call("cc_gemm", N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, epi, N.BF16, 1, N.stream_ptr())
for _ in range(3):
    run()
torch.cuda.synchronize()
lib.cc_debug_gemm_trace(ctypes.c_void_p(N.ptr(tr)))
run()
torch.cuda.synchronize()
lib.cc_debug_gemm_trace(ctypes.c_void_p(0))
t = tr.cpu().numpy()
t0 = t[:, :, 4][t[:, :, 4] > 0].min()
for c in range(148):
    row = []
    for u in range(8):
        if t[c, u, 4] == 0:
            break
        tile, o, nf, nk, a, b, e = t[c, u, :7]
        row.append(f"t{tile}o{o}/{nf}k{nk}:{(a-t0)/1e3:.1f}-{(b-t0)/1e3:.1f}-{(e-t0)/1e3:.1f}")
    print(c, " ".join(row))
