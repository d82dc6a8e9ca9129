"""Request-stream throughput through the public API with 1 vs 2 CUDA streams
(requests alternate between the streams; each request's first token is read
back after the next request has been enqueued).  Config 2."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

args = argparse.Namespace(layers=32, chunks=10, chunk_len=512, question=32, config="8b")
torch.cuda.set_device(0)
cc, model, store, chunks, question = bench.make_workload(args, 0)
r = np.random.default_rng(5)
qs = [r.integers(0, 128256, 32) for _ in range(200)]
n_prompt = 10 * 512 + 32


def stream_run(n_streams, n_req=30, warm=5):
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(n_streams - 1)]
    inflight = []
    done = []
    for i in range(n_req):
        st = streams[i % n_streams]
        with torch.cuda.stream(st):
            p = cc.build_plan(chunks, qs[i], store, alpha=1.0, cfo_override=0.15)
            res = cc.prefill(model, cc.plan_to_request(p), record_attention=False, stats=False, first_token=True)
        inflight.append(res)
        if len(inflight) > n_streams:
            _ = inflight.pop(0).first_token
            done.append(time.perf_counter())
    while inflight:
        _ = inflight.pop(0).first_token
        done.append(time.perf_counter())
    torch.cuda.synchronize()
    per = (done[-1] - done[warm - 1]) / (len(done) - warm)
    return n_prompt / per


for ns in (1, 2, 3, 4, 6, 4, 3):
    print(f"streams {ns}: {stream_run(ns):,.0f} prompt tokens/s", flush=True)
