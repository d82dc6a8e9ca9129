"""Launch-overhead probe: the config-2 fix-up step timed as stream launches
vs replayed from one CUDA graph capture (same kernels, same plan)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_15734_b200 import engine  # noqa: E402

ratio = float(sys.argv[1]) if len(sys.argv) > 1 else 0.15
args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32)
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
_, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, ratio)
last = int(np.flatnonzero(dplan.rows == req.question_span[1] - 1)[0])


def step():
    engine.execute(model, dplan, ws)
    engine._logits_rows(model, ws["hidden"][last:last + 1])


def timed(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


print("ratio", ratio, "rows", len(dplan.rows), "stream ms/step", round(timed(step), 3), flush=True)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
torch.cuda.synchronize()
print("graph  ms/step", round(timed(g.replay), 3), flush=True)
print("stream ms/step", round(timed(step), 3), flush=True)
