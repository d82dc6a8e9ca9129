"""Host-side breakdown of one e2e request (config 2): planning, request
layout, device plan upload, kernel launches, first-token readback."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_15734_b200 import engine  # noqa: E402

args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32)
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
T = {}
for rep in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = cc.build_plan(chunks, question, store, alpha=1.0, cfo_override=0.15)
    t1 = time.perf_counter()
    rq = cc.plan_to_request(p)
    t2 = time.perf_counter()
    res = cc.prefill(model, rq, record_attention=False, stats=False, first_token=True)
    tok = res.first_token
    t3 = time.perf_counter()
    if rep >= 3:
        for k, v in (("build_plan", t1 - t0), ("plan_to_request", t2 - t1), ("prefill+token", t3 - t2)):
            T.setdefault(k, []).append(v * 1e3)
for k, v in T.items():
    print(f"{k:16s} {np.median(v):8.3f} ms")
# launch-side cost of the prefill without waiting (CPU time to enqueue)
_, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, 0.15)
torch.cuda.synchronize()
t0 = time.perf_counter()
engine.execute(model, dplan, ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"execute enqueue {1e3 * (t1 - t0):.3f} ms, until done {1e3 * (t2 - t0):.3f} ms")

# where the host time before the first kernel goes (cProfile, 5 requests)
import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
for rep in range(5):
    torch.cuda.synchronize()
    pr.enable()
    p = cc.build_plan(chunks, question, store, alpha=1.0, cfo_override=0.15)
    rq = cc.plan_to_request(p)
    res = cc.prefill(model, rq, record_attention=False, stats=False, first_token=True)
    tok = res.first_token
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
