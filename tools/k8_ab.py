"""cc_segment_mass at the config-2 MISS shape (5152 stats rows, 10 chunk
segments + the question, Llama-3-8B heads), device-timed per launch."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_15734_b200 import _native as N

n, H, Hkv, dh = 5152, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((n, H * dh), generator=g, device="cuda").bfloat16()
k = torch.randn((n, Hkv * dh), generator=g, device="cuda").bfloat16()
slot = torch.arange(n, dtype=torch.int32, device="cuda")
rows = torch.arange(n, dtype=torch.int32, device="cuda")
lse = torch.full((n, H), 8.0, device="cuda")
lo = torch.tensor([i * 512 for i in range(10)] + [5120], dtype=torch.int32, device="cuda")
hi = torch.tensor([(i + 1) * 512 for i in range(10)] + [5152], dtype=torch.int32, device="cuda")
mass = torch.zeros((n, 12), dtype=torch.float64, device="cuda")


def run():
    N.call("cc_segment_mass", N.ptr(q), N.ptr(k), N.ptr(slot), None, N.ptr(lse), N.ptr(lo), N.ptr(hi), 11, N.ptr(rows),
           n, N.ptr(mass), n, H, Hkv, dh, N.BF16, N.stream_ptr())


for _ in range(3):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
fl = 2.0 * H * dh * (n * (n + 1) / 2)
print(f"segment_mass {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s  checksum {mass.sum().item():.6f}")
