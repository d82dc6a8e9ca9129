"""One bench step (config 2 fix-up prefill) inside an NVTX range "step" for
ncu: warm-up steps run outside the range.

  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_15734_b200 import engine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--ratio", type=float, default=0.15)
p.add_argument("--full", action="store_true", help="profile the full-recompute baseline step instead")
p.add_argument("--config", default="8b", choices=["8b", "8b-32k", "70b"])
a = p.parse_args()
args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32, config=a.config, tp_peer=0)
if a.config == "8b-32k":
    args.chunks = 64
elif a.config == "70b":
    args.chunks, args.chunk_len, args.layers = 16, 1024, 80
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
if a.full:
    req, dplan, ws = bench.full_plan(cc, model, chunks, question)
else:
    _, req, dplan, ws = bench.resident_plan(cc, model, store, chunks, question, a.ratio)
last = int(np.flatnonzero(dplan.rows == req.question_span[1] - 1)[0])


def step():
    engine.execute(model, dplan, ws)
    engine._logits_rows(model, ws["hidden"][last:last + 1])


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
step()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("profiled one step", flush=True)
