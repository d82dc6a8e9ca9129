"""Per-CTA timeline of the tcgen05 attention inside one config-2 step (debug):
python tools/attn_trace.py [ratio]"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_15734_b200 import _native as N, engine  # noqa: E402

ratio = float(sys.argv[1]) if len(sys.argv) > 1 else 0.15
args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32)
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
_, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, ratio)
for _ in range(2):
    engine.execute(model, dplan, ws)
torch.cuda.synchronize()
tr = torch.zeros((4096, 16), dtype=torch.int64, device="cuda")
N.lib().cc_debug_attn_trace(ctypes.c_void_p(N.ptr(tr)))
engine.execute(model, dplan, ws)
torch.cuda.synchronize()
N.lib().cc_debug_attn_trace(ctypes.c_void_p(0))
t = tr.cpu().numpy()
t = t[t[:, 1] > 0]
t0 = t[:, 1].min()
tiles, start, end, sm = t[:, 0], (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]
dur = end - start
print(f"CTAs {len(t)}  makespan {end.max():.1f} us  sum tiles {tiles.sum()}  max tiles {tiles.max()}")
print(f"per-tile us: median {np.median(dur / np.maximum(tiles, 1)):.3f}  (tiles>=20: {np.median((dur / np.maximum(tiles, 1))[tiles >= 20]):.3f})")
load = {}
for s_, d_ in zip(sm, dur):
    load[s_] = load.get(s_, 0) + d_
print(f"SMs used {len(load)}  busiest SM {max(load.values()):.1f} us  mean SM busy {np.mean(list(load.values())):.1f} us")
big = t[:, 0] >= 20
names = ["sm:s_full", "sm:p_empty2", "sm:p_empty1", "-", "mma:k_full", "mma:s_empty", "mma:p_full", "mma:v_full",
         "mma:S issue", "mma:S commit", "mma:PV issue", "mma:PV commit"]
cols = [4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15]
per = {n: np.median(t[big, c] / t[big, 0]) for n, c in zip(names, cols)}
print("stall cycles per tile (CTAs with >= 20 tiles):", {k: int(v) for k, v in per.items()})
print("cycles per tile (clock64 ~ 1.9 GHz):", int(np.median(dur[big] / t[big, 0]) * 1900))
order = np.argsort(start)
for i in order[:10]:
    print(f"  cta tiles {tiles[i]:3d} start {start[i]:6.1f} end {end[i]:6.1f} sm {sm[i]}")
for i in order[-10:]:
    print(f"  cta tiles {tiles[i]:3d} start {start[i]:6.1f} end {end[i]:6.1f} sm {sm[i]}")
