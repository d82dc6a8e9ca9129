import sys, os, numpy as np, torch, argparse, ctypes
sys.path.insert(0, ".")
import bench
from paper_2502_15734_b200 import _native as N, engine
args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32)
cc, model, store, chunks, question = bench.make_workload(args, 0)
_, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, 0.15)
for _ in range(2): engine.execute(model, dplan, ws)
torch.cuda.synchronize()
tr = torch.zeros((8192, 16), dtype=torch.int64, device="cuda")
N.lib().cc_debug_attn_trace(ctypes.c_void_p(N.ptr(tr)))
engine.execute(model, dplan, ws); torch.cuda.synchronize()
N.lib().cc_debug_attn_trace(ctypes.c_void_p(0))
t = tr.cpu().numpy(); t = t[t[:, 1] > 0]; t0 = t[:, 1].min()
st, en = (t[:, 1]-t0)/1e3, (t[:, 2]-t0)/1e3; n = t[:, 0]; dur = en - st
A = np.vstack([n, np.ones_like(n)]).T.astype(float)
coef = np.linalg.lstsq(A, dur, rcond=None)[0]
print(os.environ.get("CCB_ATTN_SPLIT"), "CTAs", len(t), "dur = %.3f us/tile * n + %.2f us" % tuple(coef), "sum dur", round(dur.sum(),0), "makespan", round(en.max(),1))
for lo, hi in [(0, 10), (10, 20), (20, 30), (30, 45)]:
    m = (n >= lo) & (n < hi)
    if m.any(): print("   tiles [%d,%d): %d CTAs, mean dur %.1f, mean start %.1f" % (lo, hi, m.sum(), dur[m].mean(), st[m].mean()))
