"""Effective cost of each kernel family inside the pipelined config-2 step
(programmatic dependent launch on): the step is timed with CUDA events with
one family's launches dropped at a time (timing only -- results are wrong).

  python tools/ablate_step.py
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_15734_b200 import _native as N, engine  # noqa: E402

args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32)
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
_, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, 0.15)
last = int(np.flatnonzero(dplan.rows == req.question_span[1] - 1)[0])
real_call = N.call
skip = set()


def call(name, *a):
    if name in skip:
        return 0
    return real_call(name, *a)


engine.N.call = call


def step():
    engine.execute(model, dplan, ws)
    engine._logits_rows(model, ws["hidden"][last:last + 1])


def timed(k=20):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = []
    for _ in range(k):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ev)


base = timed()
print(f"full step {base:.3f} ms")
for fam in (["cc_rmsnorm"], ["cc_rope_scatter_qkv"], ["cc_attention"], ["cc_gather_rope_kv"], ["cc_gemm_qkv_rope", "cc_gemm"]):
    skip.clear()
    skip.update(fam)
    t = timed()
    skip.clear()
    b2 = timed()
    print(f"without {'+'.join(fam):32s} {t:.3f} ms  -> effective {(b2 + base) / 2 - t:.3f} ms per step", flush=True)
