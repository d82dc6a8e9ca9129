"""Phase breakdown of the GPU replay (config 3 shapes, small trace)."""
import sys
import time
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_15734_b200 as cc  # noqa: E402
from paper_2502_15734_b200 import engine, planner, replay, stats, store as st_mod  # noqa: E402

T = defaultdict(float)
C = defaultdict(int)


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[name] += time.perf_counter() - t
        C[name] += 1
        return r
    setattr(mod, name, g)


for mod, name in ((replay, "build_plan"), (replay, "plan_to_request"), (replay, "prefill"), (replay, "creation_stats"),
                  (replay, "extract_chunk_cache"), (replay, "question_stream"), (replay, "predict_focused")):
    wrap(mod, name)
orig_insert = st_mod.VariantStore.insert


def ins(self, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = orig_insert(self, *a, **k)
    torch.cuda.synchronize()
    T["store.insert"] += time.perf_counter() - t
    C["store.insert"] += 1
    return r


st_mod.VariantStore.insert = ins
orig_exec = engine.execute


def ex(*a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = orig_exec(*a, **k)
    torch.cuda.synchronize()
    T["engine.execute"] += time.perf_counter() - t
    C["engine.execute"] += 1
    return r


engine.execute = ex
cfg = cc.ModelConfig.llama3_8b(dtype="bf16")
model = cc.build_model(cfg)
gen = dict(chunk_len_range=(512, 512), question_len_range=(32, 32), vocab_size=cfg.vocab_size)
tr = harness.gen_synthetic(200, 1.542, 10, 50, seed=3, **gen)
store = cc.VariantStore(cc.StoreConfig(max_chunks=100, variants_per_chunk=5))
harness.replay_gpu(tr, model, store, policy="cachecraft", warmup=0, cfo_override=0.15, measure_deviation=False,
                  records=tr.records[:20])
T.clear(), C.clear()
t0 = time.perf_counter()
rep = harness.replay_gpu(tr, model, store, policy="cachecraft", warmup=0, cfo_override=0.15, measure_deviation=False,
                        records=tr.records[20:50])
wall = time.perf_counter() - t0
print(f"30 requests wall {wall*1e3:.0f} ms; per request {wall/30*1e3:.1f} ms; ttft p50 "
      f"{np.median([r.ttft * 1e3 for r in rep.requests]):.1f} ms")
for k in sorted(T, key=lambda k: -T[k]):
    print(f"{k:22s} n={C[k]:4d} total {T[k]*1e3:8.1f} ms  per call {T[k]/C[k]*1e3:7.2f} ms")
print("hits", [r.hits for r in rep.requests])
