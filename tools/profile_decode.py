"""Decode steps of config 2 (Llama-3-8B, 5152-token fix-up context) inside an
NVTX range "decode" for ncu (graph replays included):

  ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      --clock-control none --csv --log-file gpurun_out/decode_launches.csv python tools/profile_decode.py
"""
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
res = cc.prefill(model, req, record_attention=False, stats=False)
h = torch.from_numpy(np.asarray(res.hidden[req.question_span[1] - 1], np.float64).reshape(1, -1)).cuda().float()
engine.DecodeSession(model, res.kv, 3).run(h)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("decode")
engine.DecodeSession(model, res.kv, 3).run(h)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("profiled decode", flush=True)
