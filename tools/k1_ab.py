"""K1 (cc_gather_rope_kv) A/B at the config-2 shape: register-path kernel vs the
TMA-staged bulk kernel with several column chunks.  One launch covers all 32
layers of 10 x 512 cached rows (15% of the rows recomputed: skipped).  CUDA
events on the launching stream, median of 20 launches; inputs (1.4 GB moved
per launch) are larger than L2.  Also checks that every mode writes the same
bytes.

  python tools/k1_ab.py [chunks]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_15734_b200 import _native as N  # noqa: E402

chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 10
L, kvw, dh, clen = 32, 1024, 128, 512
nb = chunks * clen // 16
n = chunks * clen + 32
g = torch.Generator(device="cuda").manual_seed(0)
pool = torch.randn((L, nb, 2, 16, kvw), device="cuda", generator=g).bfloat16()
items = np.array([(b, b * 16, 16, 0) for b in range(nb)], dtype=np.int32)
it = torch.from_numpy(items.reshape(-1)).cuda()
slot_pos = torch.arange(n, dtype=torch.int32, device="cuda")
rng = np.random.default_rng(0)
act = np.zeros(n, dtype=np.int32)
act[rng.choice(chunks * clen, int(0.15 * chunks * clen), replace=False)] = L
act[chunks * clen:] = L
active = torch.from_numpy(act).cuda()
half = dh // 2
inv = torch.from_numpy(500000.0 ** (-2.0 * np.arange(half) / dh)).cuda()
tab = torch.empty((n, half, 2), dtype=torch.float32, device="cuda")
N.call("cc_rope_table", N.ptr(tab), N.ptr(inv), n, half, N.BF16, N.stream_ptr())
bufs = [torch.zeros((L, n, kvw), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
live = int((act[: chunks * clen] == 0).sum())
alg = live * L * 5 * kvw * 2


def run():
    N.call("cc_gather_rope_kv", N.ptr(pool), pool.stride(0), pool.stride(1), N.ptr(it), len(items), 0, L,
           N.ptr(slot_pos), N.ptr(active), N.ptr(tab), *(N.ptr(b) for b in bufs), n * kvw, kvw, dh, N.BF16,
           N.stream_ptr())


ref = None
for mode in ((1, 0), (0, 0), (2, 0), (1, 0), (0, 0), (2, 0)):
    N.lib().cc_debug_k1(*mode)
    for b in bufs:
        b.zero_()
    run()
    torch.cuda.synchronize()
    sig = [b.view(torch.int16).to(torch.int64).sum().item() for b in bufs]
    if ref is None:
        ref = [b.clone() for b in bufs]
    same = all(torch.equal(a, b) for a, b in zip(ref, bufs))
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(23):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts[3:]))
    print(f"mode ldg={mode[0]} cols={mode[1]:4d}: {us:8.1f} us  {alg / us / 1e3:7.1f} GB/s  identical={same} sig={sig[0]}")
