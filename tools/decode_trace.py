"""Timeline of the decode chain (config 2: Llama-3-8B shapes, 5.2k-token
fix-up context) from the in-kernel %globaltimer records
(cc_debug_decode_trace): per launch of the GEMV / fused-attention kernels,
start (first CTA), wait released, end (last CTA), CTAs per SM.

  python tools/decode_trace.py [n_layers_to_print]
"""
import argparse
import collections
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_15734_b200 import _native as N  # noqa: E402
from paper_2502_15734_b200 import engine  # noqa: E402

show = int(sys.argv[1]) if len(sys.argv) > 1 else 3
args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32)
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
_, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, 0.15)
res = cc.prefill(model, req, record_attention=False, stats=False)
h = torch.from_numpy(np.asarray(res.hidden[req.question_span[1] - 1], np.float64).reshape(1, -1)).cuda().float()
engine.DecodeSession(model, res.kv, 3).run(h)
torch.cuda.synchronize()
cap = 400000
buf = torch.zeros((cap, 8), dtype=torch.int64, device="cuda")
lib = N.lib()
lib.cc_debug_decode_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
sess = engine.DecodeSession(model, res.kv, 3)
lib.cc_debug_decode_trace(ctypes.c_void_p(buf.data_ptr()), cap)
sess.run(h)
torch.cuda.synchronize()
lib.cc_debug_decode_trace(None, 0)
r = buf.cpu().numpy().astype(np.uint64)
r = r[r[:, 3] != 0]
tag = (r[:, 3] >> np.uint64(48)).astype(int)
tag[tag == 4] = 3
sm = ((r[:, 3] >> np.uint64(32)) & np.uint64(0xFFFF)).astype(int)
blk = (r[:, 3] & np.uint64(0xFFFFFFFF)).astype(int)
t0, t1, t2 = (r[:, i].astype(np.int64) for i in range(3))
cps = r[:, 4:8].astype(np.int64)
order = np.argsort(t0, kind="stable")
launches = []
cur = {}
for i in order:
    k = tag[i]
    L = cur.get(k)
    if L is None or blk[i] in L["blk"]:
        L = {"tag": k, "blk": set(), "idx": []}
        cur[k] = L
        launches.append(L)
    L["blk"].add(blk[i])
    L["idx"].append(i)
launches.sort(key=lambda L: t0[L["idx"]].min())
base = t0.min()
names = {1: "gemv_stream", 2: "gemv_rows", 3: "attn_fused"}
print(f"{len(r)} CTA records, {len(launches)} launches; globaltimer distinct deltas (ns):",
      np.unique(np.diff(np.sort(t0)))[:8])
prev_end = None
rows = []
for L in launches:
    ix = np.array(L["idx"])
    per_sm = collections.Counter(sm[ix])
    a, w0, w1, e = t0[ix].min(), t1[ix].min(), t1[ix].max(), t2[ix].max()
    rows.append((names[L["tag"]], len(ix), len(per_sm), max(per_sm.values()), a - base, w0 - base, w1 - base, e - base,
                 np.median(t2[ix] - t1[ix])))
# steady state: the middle third of the launches
n = len(rows)
print(f"{'kernel':12s} {'CTAs':>5s} {'SMs':>4s} {'max/SM':>6s} {'start':>9s} {'wait0':>9s} {'wait1':>9s} {'end':>9s} "
      f"{'dur':>7s} {'gap':>6s} {'med_cta':>7s}")
lo = n // 2
for i in range(lo, min(n, lo + 5 * show)):
    nm, c, s, mx, a, w0, w1, e, med = rows[i]
    gap = (w0 - rows[i - 1][7]) if i else 0
    print(f"{nm:12s} {c:5d} {s:4d} {mx:6d} {a/1e3:9.2f} {w0/1e3:9.2f} {w1/1e3:9.2f} {e/1e3:9.2f} {(e - w0)/1e3:7.2f} "
          f"{gap/1e3:6.2f} {med/1e3:7.2f}")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for i in range(n // 3, 2 * n // 3):
    nm, c, s, mx, a, w0, w1, e, med = rows[i]
    tot[nm] += (e - w0) / 1e3
    cnt[nm] += 1
print("mean wait-released -> end (us):", {k: round(tot[k] / cnt[k], 2) for k in tot})
# streaming GEMV checkpoints per launch in the middle third: prologue (x staged), loop end (before the CTA barrier)
gl = [L for L in launches if L["tag"] == 1]
if gl:
    k = len(gl) // 2
    for L in gl[k:k + 4]:
        ix = np.array(L["idx"])
        c = cps[ix] / 1e3
        print("gemv_stream launch: row landed %.2f, reduced %.2f, x staged %.2f, loop done %.2f (median), %.2f (max), "
              "CTA end %.2f (median) us after release"
              % (np.median(c[:, 2]), np.median(c[:, 3]), np.median(c[:, 0]), np.median(c[:, 1]), c[:, 1].max(),
                 np.median((t2 - t1)[ix]) / 1e3))
att = (tag == 3) & (cps[:, 0] > 0)
if att.any():
    c = cps[att] / 1e3
    last = (r[:, 3] >> np.uint64(48)).astype(int)[att] == 4
    print("attention CTA checkpoints after release (us, median): rope/append/fix %.2f, steps %.2f, merge+partial+ticket %.2f, end %.2f"
          % (np.median(c[:, 0]), np.median(c[:, 1]), np.median(c[:, 2]), np.median((t2 - t1)[att]) / 1e3))
    if last.any():
        print("combining CTAs: ticket at %.2f, end %.2f" % (np.median(c[last, 2]), np.median((t2 - t1)[att][last]) / 1e3))
