"""cc_gemv (M = 1) bandwidth over shapes: is the down projection's 4.6 TB/s a
shape (row length / output count) effect?  Weights rotate over copies > L2."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_15734_b200 import _native as N

N.lib().cc_set_pdl(1)


def timeit(fn, reps=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


shapes = [(4096, 14336, N.EPI_RESID_ADD), (4096, 14336, N.EPI_STORE), (4096, 16384, N.EPI_RESID_ADD),
          (4096, 12288, N.EPI_RESID_ADD), (14336, 4096, N.EPI_RESID_ADD), (8192, 8192, N.EPI_RESID_ADD),
          (2048, 28672, N.EPI_RESID_ADD), (16384, 4096, N.EPI_STORE), (28672, 4096, N.EPI_SWIGLU)]
for Nn, K, epi in shapes:
    nb = Nn * K * 2
    Ws = [(torch.randn((Nn, K), device="cuda") / 64).bfloat16() for _ in range(max(2, int(6e8 // nb)))]
    A = torch.randn((1, K), device="cuda").bfloat16()
    C = torch.zeros((1, Nn), device="cuda") if epi == N.EPI_RESID_ADD else torch.empty(
        (1, Nn // 2 if epi == N.EPI_SWIGLU else Nn), device="cuda", dtype=torch.bfloat16)
    it = [0]

    def run():
        W = Ws[it[0] % len(Ws)]
        it[0] += 1
        N.call("cc_gemv", N.ptr(A), K, N.ptr(W), K, N.ptr(C), C.shape[1], 1, Nn, K, epi, N.stream_ptr())

    ms = timeit(run)
    print(f"N={Nn:6d} K={K:6d} epi={epi}: {ms*1e3:7.1f} us  {nb/1e9/ms*1e3:7.0f} GB/s", flush=True)
    del Ws
