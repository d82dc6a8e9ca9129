"""Decode building blocks at Llama-3-8B shapes: cc_gemv per projection (M=1)
and cc_decode_attention over n keys, device-timed; GB/s vs HBM."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_15734_b200 import _native as N

import os

if os.environ.get("CCB_BENCH_PDL") == "1":  # chained launches overlap (the decode chain's mode)
    N.lib().cc_set_pdl(1)

shapes = [("qkv", 6144, 4096, N.EPI_STORE), ("o", 4096, 4096, N.EPI_RESID_ADD), ("gate_up", 28672, 4096, N.EPI_SWIGLU),
          ("down", 4096, 14336, N.EPI_RESID_ADD), ("unembed-like", 128256, 4096, N.EPI_STORE)]


def timeit(fn, reps=50):
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


# weights > L2 in aggregate: rotate over 8 copies so each call streams from HBM
for name, Nn, K, epi in shapes:
    Ws = [(torch.randn((Nn, K), device="cuda") / 64).bfloat16() for _ in range(4 if Nn > 100000 else 8)]
    A = torch.randn((1, K), device="cuda").bfloat16()
    C = torch.zeros((1, Nn), device="cuda") if epi == N.EPI_RESID_ADD else torch.empty(
        (1, Nn // 2 if epi == N.EPI_SWIGLU else Nn), device="cuda", dtype=torch.bfloat16)
    it = [0]

    def run():
        W = Ws[it[0] % len(Ws)]
        it[0] += 1
        N.call("cc_gemv", N.ptr(A), K, N.ptr(W), K, N.ptr(C), C.shape[1], 1, Nn, K, epi, N.stream_ptr())

    ms = timeit(run)
    gb = Nn * K * 2 / 1e9
    print(f"gemv {name:12s} N={Nn:6d} K={K:6d}: {ms*1e3:7.1f} us  {gb/ms*1e3:7.0f} GB/s", flush=True)
    del Ws

for n in (() if os.environ.get("CCB_BENCH_NOATTN") else (1024, 5152, 32800)):
    Hq, Hkv, dh = 32, 8, 128
    q = torch.randn((Hq * dh,), device="cuda").bfloat16()
    ks = [torch.randn((n, Hkv * dh), device="cuda").bfloat16() for _ in range(4)]
    v = torch.randn((n, Hkv * dh), device="cuda").bfloat16()
    ctx = torch.empty((Hq * dh,), device="cuda", dtype=torch.bfloat16)
    lse = torch.empty((Hq,), device="cuda")
    it = [0]

    def run():
        k = ks[it[0] % 4]
        it[0] += 1
        N.call("cc_decode_attention", N.ptr(q), N.ptr(k), N.ptr(v), None, N.ptr(ctx), N.ptr(lse), n, Hq, Hkv, dh,
               N.stream_ptr())

    ms = timeit(run)
    gb = 2 * n * Hkv * dh * 2 / 1e9
    print(f"decode_attention n={n:6d}: {ms*1e3:7.1f} us  {gb/ms*1e3:7.0f} GB/s", flush=True)
