"""Steady-state replay requests inside NVTX range "req" (for an ncu launch list)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2502_15734_b200 as cc  # noqa: E402
from paper_2502_15734_b200 import harness  # noqa: E402

cfg = cc.ModelConfig.llama3_8b(dtype="bf16")
model = cc.build_model(cfg)
gen = dict(chunk_len_range=(512, 512), question_len_range=(32, 32), vocab_size=cfg.vocab_size)
tr = harness.gen_synthetic(200, 1.542, 10, 40, seed=3, **gen)
store = cc.VariantStore(cc.StoreConfig(max_chunks=100, variants_per_chunk=5))
harness.replay_gpu(tr, model, store, policy="cachecraft", warmup=0, cfo_override=0.15, measure_deviation=False,
                  records=tr.records[:30])
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("req")
t0 = time.perf_counter()
rep = harness.replay_gpu(tr, model, store, policy="cachecraft", warmup=0, cfo_override=0.15, measure_deviation=False,
                        records=tr.records[30:33])
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) * 1e3, "hits", [r.hits for r in rep.requests],
      "computed", [r.tokens_computed for r in rep.requests], "token_layers", [r.token_layers for r in rep.requests])
torch.cuda.nvtx.range_pop()
