"""Per-CTA timeline of the ping-pong attention kernel (variant 4) on the
attn_ab.py cases (debug):  python tools/attn_pp_trace.py [case-substring] [variant]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import attn_ab  # noqa: E402
from paper_2502_15734_b200 import _native as N  # noqa: E402

sel = sys.argv[1] if len(sys.argv) > 1 else "r=.15"
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 4
lib = N.lib()
lib.cc_debug_attn_variant(variant)
for name, (n_q, n, Hq, Hkv) in attn_ab.CASES.items():
    if sel not in name:
        continue
    args = attn_ab.make(n_q, n, Hq, Hkv)
    ctx = torch.empty((n_q, Hq * 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((n_q, Hq), dtype=torch.float32, device="cuda")
    for _ in range(3):
        attn_ab.run(args, ctx, lse)
    torch.cuda.synchronize()
    W = 24 if variant in (4, 5) else 16
    tr = torch.zeros((8192, W), dtype=torch.int64, device="cuda")
    lib.cc_debug_attn_trace(ctypes.c_void_p(N.ptr(tr)))
    attn_ab.run(args, ctx, lse)
    torch.cuda.synchronize()
    lib.cc_debug_attn_trace(ctypes.c_void_p(0))
    t = tr.cpu().numpy()
    t = t[t[:, 1] > 0]
    t0 = t[:, 1].min()
    tiles, start, end, sm = t[:, 0], (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]
    dur = end - start
    print(f"== {name}: CTAs {len(t)}  makespan {end.max():.1f} us  sum tiles {tiles.sum()}  max tiles {tiles.max()}")
    load = {}
    for s_, d_ in zip(sm, dur):
        load[s_] = load.get(s_, 0) + d_
    print(f"SMs used {len(load)}  busiest SM {max(load.values()):.1f} us  mean SM busy {np.mean(list(load.values())):.1f} us")
    big = tiles >= 1
    per = lambda c: int(np.median(t[big, c] / t[big, 0]))  # noqa: E731
    print(f"us per tile-pair (median, big CTAs): {np.median(dur[big] / tiles[big]):.3f}")
    print("cycles per tile-pair: sm0 s_full wait", per(4), "busy", per(5), "epilogue", per(6),
          "| sm1 s_full wait", per(7), "busy", per(8), "epilogue", per(9),
          "| mma p_full wait", per(10), "other waits", per(11), "| tma q_empty", per(12), "k/v_empty", per(13),
          "| sm0 o_done wait", per(14), "merge", per(15))
    print("totals per CTA (median cycles): sm0 wait", int(np.median(t[:, 4])), "busy", int(np.median(t[:, 5])),
          "epi", int(np.median(t[:, 6])), "o_done", int(np.median(t[:, 14])), "split-epi", int(np.median(t[:, 15])))
    if t.shape[1] > 16:
        print("mma thread per tile: commit", per(16), "issue", per(17))
    if False:
        print("split epilogue totals (sum over CTAs / count): ticket", int(t[:, 16].sum() / max(1, (t[:, 19] + t[:, 20]).sum())),
              "park", int(t[:, 17].sum() / max(1, t[:, 19].sum())), "merge", int(t[:, 18].sum() / max(1, t[:, 20].sum())),
              "parks", int(t[:, 19].sum()), "merges", int(t[:, 20].sum()))
        nm = max(1, t[:, 20].sum())
        print("merge detail per merge: to fence", int(t[:, 21].sum() / nm), "(xbar+fence", int(t[:, 22].sum() / nm),
              ") ml loads", int(t[:, 23].sum() / nm))
    order = np.argsort(start)
    for i in list(order[:4]) + list(order[-6:]):
        print(f"  cta tiles {tiles[i]:3d} start {start[i]:6.1f} end {end[i]:6.1f} dur {dur[i]:6.1f} sm {sm[i]}")
    longest = np.argsort(-dur)[:5]
    for i in longest:
        print(f"  long: tiles {tiles[i]:3d} start {start[i]:6.1f} dur {dur[i]:6.1f} us/tile {dur[i] / max(tiles[i], 1):.3f}")
lib.cc_debug_attn_variant(-1)
