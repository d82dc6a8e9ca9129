"""Config-2 fix-up step device time (CUDA events, 20 steps) with programmatic
dependent launch on and off, alternating, same process."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_15734_b200 import engine  # noqa: E402

args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32)
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
_, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, 0.15)
last = int(np.flatnonzero(dplan.rows == req.question_span[1] - 1)[0])


def step():
    engine.execute(model, dplan, ws)
    engine._logits_rows(model, ws["hidden"][last:last + 1])


def timed(k=20):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


ref = None
for rep in range(3):
    for pdl in (False, True):
        model.prefill_pdl = pdl
        ms = timed()
        out = ws["hidden"].float().clone()
        if ref is None:
            ref = out
        print(f"pdl={int(pdl)} ms/step {ms:.3f} same_bits={torch.equal(out, ref)}", flush=True)
