"""Per-shape GEMM timing: our tcgen05 kernel vs torch.matmul (cuBLAS), bf16."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_15734_b200 import _native as N

shapes = [("qkv", 6144, 4096, N.EPI_STORE), ("o", 4096, 4096, N.EPI_RESID_ADD), ("gate_up", 28672, 4096, N.EPI_SWIGLU),
          ("down", 4096, 14336, N.EPI_RESID_ADD)]
Ms = [int(x) for x in sys.argv[1:]] or [802, 5152]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for M in Ms:
    for name, Nn, K, epi in shapes:
        A = torch.randn((M, K), device="cuda").bfloat16()
        B = (torch.randn((Nn, K), device="cuda") / 64).bfloat16()
        if epi == N.EPI_RESID_ADD:
            C = torch.zeros((M, Nn), device="cuda")
        elif epi == N.EPI_SWIGLU:
            C = torch.empty((M, Nn // 2), device="cuda", dtype=torch.bfloat16)
        else:
            C = torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)
        ours = timeit(lambda: N.call("cc_gemm", N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, epi, N.BF16,
                                     1, N.stream_ptr()))
        ref = timeit(lambda: torch.matmul(A, B.T))
        fl = 2.0 * M * Nn * K
        print(f"M={M:5d} {name:8s} N={Nn:6d} K={K:6d}: ours {ours*1e3:8.1f} us {fl/ours/1e9:7.1f} TF/s | "
              f"cuBLAS {ref*1e3:8.1f} us {fl/ref/1e9:7.1f} TF/s | ratio {ref/ours:5.2f}", flush=True)
