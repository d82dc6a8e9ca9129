"""A/B: fused QKV GEMM + RoPE + scatter (cc_gemm_qkv_rope) vs cc_gemm + cc_rope_scatter_qkv
at the config-2 shape (CUDA events, median of 50)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_15734_b200 import _native as N  # noqa: E402

for M in (290, 802, 1570, 5152):
    Hq, Hkv, d, dh, n_slots = 32, 8, 4096, 128, 5152
    NQ = (Hq + 2 * Hkv) * dh
    x = torch.randn((M, d), device="cuda").bfloat16()
    w = (torch.randn((NQ, d), device="cuda") / 64).bfloat16()
    slots = torch.sort(torch.randperm(n_slots, device="cuda")[:M]).values.int()
    pos = slots.clone()
    table = torch.randn((n_slots, 64, 2), device="cuda")
    q = torch.empty((M, Hq * dh), dtype=torch.bfloat16, device="cuda")
    kk, vv, kr = [torch.empty((n_slots, Hkv * dh), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    qkv = torch.empty((M, NQ), dtype=torch.bfloat16, device="cuda")
    s = N.stream_ptr()

    def fused():
        N.call("cc_gemm_qkv_rope", N.ptr(x), d, N.ptr(w), d, M, d, N.ptr(slots), N.ptr(pos), N.ptr(table), N.ptr(q),
               N.ptr(kk), N.ptr(vv), N.ptr(kr), N.ptr(qkv), Hq, Hkv, dh, N.BF16, s)

    def unfused():
        N.call("cc_gemm", N.ptr(x), d, N.ptr(w), d, N.ptr(qkv), NQ, M, NQ, d, N.EPI_STORE, N.BF16, 0, s)
        N.call("cc_rope_scatter_qkv", N.ptr(qkv), NQ, M, N.ptr(slots), N.ptr(pos), N.ptr(table), N.ptr(q), N.ptr(kk),
               N.ptr(vv), N.ptr(kr), Hq, Hkv, dh, N.BF16, s)

    out = []
    for name, f in (("fused", fused), ("gemm+rope_scatter", unfused)):
        for _ in range(5):
            f()
        ev = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        out.append(f"{name} {statistics.median(x.elapsed_time(y) for x, y in ev) * 1e3:7.1f} us")
    print(f"M={M}: " + " | ".join(out), flush=True)
