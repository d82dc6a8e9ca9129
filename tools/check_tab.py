"""Correctness + timing of the unit-table swap GEMM against the fp32 reference
and against the data-parallel tiling (bitwise).  Run with CCB_GEMM_FORCE unset;
each mode runs in a subprocess (the force variable is read once)."""
import os
import subprocess
import sys

CODE = r"""
import math, sys, torch
sys.path.insert(0, '.')
from paper_2502_15734_b200 import _native as N
M, Nn, K, epi = {M}, {Nn}, {K}, '{epi}'
g = torch.Generator(device='cuda').manual_seed(11)
A = torch.randn((M, K), generator=g, device='cuda').bfloat16()
B = (torch.randn((Nn, K), generator=g, device='cuda') / math.sqrt(K)).bfloat16()
acc = A.float() @ B.float().T
code = dict(store=N.EPI_STORE, resid=N.EPI_RESID_ADD, swiglu=N.EPI_SWIGLU, gelu=N.EPI_GELU)[epi]
def run():
    if epi == 'resid':
        C = torch.ones((M, Nn), device='cuda')
    elif epi == 'swiglu':
        C = torch.empty((M, Nn // 2), device='cuda', dtype=torch.bfloat16)
    else:
        C = torch.empty((M, Nn), device='cuda', dtype=torch.bfloat16)
    N.call('cc_gemm', N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, code, N.BF16, 4, N.stream_ptr())
    return C
C = run()
if epi == 'resid': ref = acc + 1
elif epi == 'swiglu':
    a4 = acc.reshape(M, Nn // 128, 2, 64); ref = (torch.nn.functional.silu(a4[:, :, 0]) * a4[:, :, 1]).reshape(M, Nn // 2)
elif epi == 'gelu': ref = torch.nn.functional.gelu(acc, approximate='tanh')
else: ref = acc
err = ((C.float() - ref).abs() / (ref.abs() + 1e-2)).max().item()
torch.save(C.cpu(), '/tmp/ct_{tag}.pt')
for _ in range(3): run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): run()
b.record(); torch.cuda.synchronize()
us = a.elapsed_time(b) / 20 * 1e3
print(f"RESULT maxrel={{err:.3g}} us={{us:.1f}} tf={{2*M*Nn*K/us/1e6:.0f}}")
"""

shapes = [(802, 6144, 4096, "store"), (802, 4096, 4096, "resid"), (802, 28672, 4096, "swiglu"),
          (802, 4096, 14336, "resid"), (300, 1536, 1024, "gelu"), (37, 1536, 1024, "store"), (1, 512, 256, "store"),
          (2048, 1024, 512, "swiglu")]
for M, Nn, K, epi in shapes:
    res = {}
    for mode in ["auto", "256,0", "0,4"]:
        env = dict(os.environ)
        env.pop("CCB_GEMM_FORCE", None)
        if mode != "auto":
            env["CCB_GEMM_FORCE"] = mode
        tag = mode.replace(",", "_")
        out = subprocess.run([sys.executable, "-c", CODE.format(M=M, Nn=Nn, K=K, epi=epi, tag=tag)], env=env,
                             capture_output=True, text=True, timeout=300)
        line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
        res[mode] = line[0][7:] if line else "FAIL " + out.stderr[-300:]
    import torch
    same = "?"
    try:
        same = torch.equal(torch.load("/tmp/ct_256_0.pt"), torch.load("/tmp/ct_0_4.pt"))
    except Exception as e:  # noqa
        same = f"n/a ({e})"[:40]
    print(f"M={M} N={Nn} K={K} {epi}: " + " | ".join(f"{k}: {v}" for k, v in res.items()) + f" | pair==dp bits: {same}",
          flush=True)
