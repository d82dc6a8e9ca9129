"""Benchmark: Cache-Craft chunk-cache fix-up prefill on B200.

Metric (BASELINE.json): prefill tokens/s and p50 TTFT at 15% recompute vs
full recompute.  Workload (BASELINE config 2): Llama-3-8B shapes (L=32,
d=4096, 32 q / 8 kv heads, SwiGLU 14336, vocab 128256, theta 5e5), random
init bf16, 10 retrieved chunks x 512 tokens + 32-token question, every chunk
a HIT whose recompute set (77 tokens = 15%) is chosen by the K9 top-k kernel
from its variant's token scores.  A "step" = one fix-up prefill of that
request through the greedy first token.

  value  device-timed (CUDA events, inputs resident in HBM) prompt tokens/s
  e2e    the same through the public API (build_plan -> plan_to_request ->
         prefill(first_token=True)) with host token lists, H2D of the layout
         and D2H of the selections / first token inside the timed region.

Usage: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Under torchrun each rank serves its own request stream (request-sharded,
no data-path collective): value = sum of per-rank tokens / max-rank time.
"""

from __future__ import annotations

import argparse
import contextlib
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill tokens/sec at 15% recompute (Llama-3-8B shapes, 10x512+32)"
WORKLOADS = {
    "8b": "config2: Llama-3-8B shapes, 1 request of 10x512 reused chunks + 32-token question, 15% recompute per "
          "chunk (K9 top-k of variant token scores)",
    "8b-32k": "config5: Llama-3-8B shapes, 32k prompt of 64x512 reused chunks + 32, 15% recompute",
    "70b": "config4: Llama-3-70B shapes, 16x1024 reused chunks + 32, 15% recompute, head-sharded TP{world}",
}
MODELS = {
    "8b": "Llama-3-8B-shaped (L=32,d=4096,Hq=32,Hkv=8,dh=128,ff=14336,vocab=128256)",
    "8b-32k": "Llama-3-8B-shaped (L=32,d=4096,Hq=32,Hkv=8,dh=128,ff=14336,vocab=128256)",
    "70b": "Llama-3-70B-shaped (L=80,d=8192,Hq=64,Hkv=8,dh=128,ff=28672,vocab=128256)",
}
UNIT = "tokens/s"


def recompute_count(n: int, cfo: float) -> int:
    """planner.py:30 (host float64) — shared by both arms' config."""
    return min(n, int(math.ceil(cfo * n - 1e-9))) if cfo > 0 else 0


def workload_config(args, world: int) -> dict:
    """The workload description, identical in both arms (computed from the
    arguments only, no package objects)."""
    tp_mode = args.config == "70b" and world > 1
    return {"workload": WORKLOADS[args.config].format(world=world),
            "model": MODELS[args.config],
            "layers": args.layers, "chunks": args.chunks, "chunk_len": args.chunk_len,
            "question": args.question, "recompute_ratio": args.ratio,
            "prompt_tokens": args.chunks * args.chunk_len + args.question,
            "recomputed_rows": args.chunks * recompute_count(args.chunk_len, args.ratio) + args.question,
            "parallelism": f"tensor-parallel x{world}" if tp_mode else f"request-sharded x{world}",
            "l2": "inputs larger than L2 (%s GB of weights streamed per step)" % (
                "140" if args.config == "70b" else "16")}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--ratio", type=float, default=0.15)
    p.add_argument("--streams", type=int, default=-1,
                   help="requests in flight on as many CUDA streams (serving mode; -1: 6 for 8b, 2 for 8b-32k, 1 for 70b)")
    p.add_argument("--layers", type=int, default=32)
    p.add_argument("--chunks", type=int, default=10)
    p.add_argument("--chunk-len", type=int, default=512)
    p.add_argument("--question", type=int, default=32)
    p.add_argument("--sweep", action="store_true", help="also report the recompute-ratio sweep 0..50%%")
    p.add_argument("--no-baselines", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--tp-peer", type=int, default=0,
                   help="70b TP: fused push-GEMM + peer-memory reduction instead of NCCL all-reduce")
    p.add_argument("--tiers", type=int, default=1, help="time the host-tier (f2) variant of the fix-up; 0 skips")
    p.add_argument("--decode-steps", type=int, default=32,
                   help="greedy decode tokens timed after the fix-up (SURVEY f3); 0 skips")
    p.add_argument("--cpu-layers", type=int, default=2, help="layers in the bounded CPU-oracle sample")
    p.add_argument("--requests", type=int, default=60, help="zipf: trace length (per rank before sharding x world)")
    p.add_argument("--config", default="8b", choices=["8b", "8b-32k", "70b", "zipf"],
                   help="8b = BASELINE config 2 (default); 8b-32k = config 5 (64x512+32); "
                        "70b = config 4 (Llama-3-70B shapes, 16x1024+32, tensor parallel over the ranks); "
                        "zipf = config 3 (Zipf trace replay, request-sharded)")
    a = p.parse_args()
    if a.config == "8b-32k":
        a.chunks = 64
    elif a.config == "70b":
        a.chunks, a.chunk_len = 16, 1024
        if a.layers == 32:
            a.layers = 80
    return a


# ---------------------------------------------------------------------------
# distributed plumbing (barrier + max-over-ranks timing only)
# ---------------------------------------------------------------------------


def dist_init(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world


def barrier(world):
    import torch

    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------


def make_workload(args, rank):
    """Model + store with one variant per chunk (created by a fresh prefill of
    the chunks in another order) + the fix-up request's host inputs."""
    import torch

    import paper_2502_15734_b200 as cc

    tp = None
    if getattr(args, "config", "8b") == "70b":
        from paper_2502_15734_b200 import parallel

        cfg = cc.ModelConfig.llama3_70b(n_layers=args.layers, dtype="bf16", seed=0)
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world > 1:
            peer = None
            if getattr(args, "tp_peer", 0):
                # fused push-GEMM + peer-memory reduction over NVLink (CUDA IPC buffers)
                m_cap = -(-int(args.chunks * args.chunk_len * 0.2 + args.question + 128) // 128) * 128
                peer = parallel.PeerComm.over_ipc(rank, world, cfg.d_model, m_cap, torch.device("cuda", rank))
            tp = parallel.TPContext(parallel.tp_slices(cfg.n_heads, cfg.kv_heads(), cfg.ff_dim(), rank, world),
                                    peer=peer)
        model = cc.build_model(cfg, tp=tp)
        r = np.random.default_rng(1000)  # every TP rank serves the same request
    else:
        cfg = cc.ModelConfig.llama3_8b(n_layers=args.layers, dtype="bf16", seed=0)
        model = cc.build_model(cfg)
        r = np.random.default_rng(1000 + rank)
    chunks = [r.integers(0, cfg.vocab_size, args.chunk_len) for _ in range(args.chunks)]
    question = r.integers(0, cfg.vocab_size, args.question)
    store = cc.VariantStore(cc.StoreConfig(max_chunks=max(100, args.chunks), variants_per_chunk=5))
    # creation: chunks prefilled fresh in a rotated order (so the fix-up's prefixes differ)
    rot = chunks[1:] + chunks[:1]
    req0 = cc.plain_request(*rot, [])
    res0 = cc.prefill(model, req0, record_attention=False, stats=False)
    ids = [cc.chunk_hash(c) for c in rot]
    for i, (s, e) in enumerate(req0.segment_slots):
        cache = cc.extract_chunk_cache(res0, s, e, source_prefix=tuple(ids[:i]))
        # token scores: synthetic (seeded) — selection cost/shape is what the bench measures
        scores = r.standard_normal(e - s)
        prefix = cc.PrefixContext(chunk_ids=tuple(ids[:i]), weights=tuple(1.0 for _ in ids[:i]))
        store.insert(ids[i], prefix=prefix, a_bar=0.1, b_bar=0.02, cci=cc.cci(0.1, 0.02), token_scores=scores,
                     cache=cache)
    del res0
    torch.cuda.synchronize()
    return cc, model, store, chunks, question


def resident_plan(cc, model, store, chunks, question, ratio):
    """Plan + device layout for the value timing (inputs resident)."""
    from paper_2502_15734_b200 import engine

    plan = cc.build_plan(chunks, question, store, alpha=1.0, cfo_override=ratio)
    req = cc.plan_to_request(plan)
    payloads = engine._payloads(model, req)
    dplan = engine.DevicePlan(model, req.token_ids, req.positions, req.is_pad, req.recompute_mask,
                              req.recompute_depth, req.segment_slots, payloads, req.question_span)
    ws = engine._workspace(model, dplan)
    return plan, req, dplan, ws


def full_plan(cc, model, chunks, question):
    from paper_2502_15734_b200 import engine

    req = cc.plain_request(*chunks, question)
    dplan = engine.DevicePlan(model, req.token_ids, req.positions, req.is_pad, req.recompute_mask,
                              req.recompute_depth, req.segment_slots, [None] * len(chunks), req.question_span)
    return req, dplan, engine._workspace(model, dplan)


def prefix_plan(cc, model, store, chunks, question, hit_chunks):
    """Prefix caching: the first `hit_chunks` chunks reused verbatim (exact
    prefix, nothing recomputed), the rest computed fresh (harness.py:512-550)."""
    from paper_2502_15734_b200 import engine

    segs = []
    for i, c in enumerate(chunks):
        if i < hit_chunks:
            v = store.lookup(cc.chunk_hash(c))[0]
            segs.append(cc.Segment(tokens=c, cache=v.cache))
        else:
            segs.append(cc.Segment(tokens=c))
    req = cc.build_request(segs, question)
    payloads = engine._payloads(model, req)
    dplan = engine.DevicePlan(model, req.token_ids, req.positions, req.is_pad, req.recompute_mask,
                              req.recompute_depth, req.segment_slots, payloads, req.question_span)
    return req, dplan, engine._workspace(model, dplan)


def time_device(model, dplan, ws, req, steps, warmup, world, timer_steps=0):
    """Device time per step (ms) with CUDA events; returns (ms list, KernelTimer)."""
    import torch

    from paper_2502_15734_b200 import engine

    q1 = req.question_span[1]
    last_row = int(np.flatnonzero(dplan.rows == q1 - 1)[0])

    def step(timer=None):
        engine.execute(model, dplan, ws, timer=timer)
        engine._logits_rows(model, ws["hidden"][last_row:last_row + 1])

    for _ in range(warmup):
        step()
    barrier(world)
    times = []
    timer = engine.KernelTimer() if timer_steps else None
    for i in range(steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        step(timer if i >= steps - timer_steps else None)  # (instrumented steps last)
        b.record()
        times.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in times]
    return ms, timer


def time_device_streams(model, runs, steps, warmup, world):
    """Serving throughput with inputs resident: ``runs`` = one (dplan, ws,
    req) per CUDA stream, each stream replaying its own request; the timed
    region spans every stream (start event on the main stream, all streams
    wait on it; the main stream waits on every stream's end event).
    Returns the device ms per request (amortised over all streams)."""
    import torch

    from paper_2502_15734_b200 import engine

    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in runs]
    rows = [int(np.flatnonzero(dp.rows == rq.question_span[1] - 1)[0]) for dp, _, rq in runs]

    def burst(n):
        for _ in range(n):
            for (dp, ws, _), st, r in zip(runs, streams, rows):
                with torch.cuda.stream(st):
                    engine.execute(model, dp, ws)
                    engine._logits_rows(model, ws["hidden"][r:r + 1])

    with engine.concurrent_streams():
        for st in streams:
            st.wait_stream(main)
        burst(warmup)
        for st in streams:
            main.wait_stream(st)
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        for st in streams:
            st.wait_event(a)
        burst(steps)
        for st in streams:
            main.wait_stream(st)
        b.record(main)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / (steps * len(runs))


def torch_reference_full(model, tokens):
    """Library baseline for full recompute: cuBLAS GEMMs (torch.matmul bf16)
    + cuDNN fused attention (torch SDPA's cuDNN backend, Blackwell-native;
    flash_attn 2.8 only if cuDNN is unavailable).  Same weights, same math;
    not our kernels."""
    import torch
    import torch.nn.functional as F

    cfg = model.config
    H, Hkv, dh, d, ff = cfg.n_heads, cfg.kv_heads(), cfg.head_dim(), cfg.d_model, cfg.ff_dim()
    n = tokens.numel()
    pos = torch.arange(n, device="cuda", dtype=torch.float64)
    inv = torch.from_numpy(cfg.rpe_base ** (-2.0 * np.arange(dh // 2) / dh)).cuda()
    ang = pos[:, None] * inv[None, :]
    cos, sin = torch.cos(ang).float(), torch.sin(ang).float()

    def rope(x):  # x [n, h, dh]
        a, b = x[..., : dh // 2].float(), x[..., dh // 2:].float()
        c, s = cos[:, None, :], sin[:, None, :]
        return torch.cat([a * c - b * s, a * s + b * c], dim=-1).bfloat16()

    from torch.nn.attention import SDPBackend, sdpa_kernel

    group = H // Hkv

    def attn_cudnn(q, k, v):  # cuDNN's Blackwell fused attention (sm_100 kernels)
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            o = F.scaled_dot_product_attention(q.transpose(0, 1)[None],
                                               k.repeat_interleave(group, dim=1).transpose(0, 1)[None],
                                               v.repeat_interleave(group, dim=1).transpose(0, 1)[None],
                                               is_causal=True)
        return o[0].transpose(0, 1)

    def attn_flash(q, k, v):  # flash_attn 2.8 (sm_80-class kernels on sm_100)
        from flash_attn import flash_attn_func

        return flash_attn_func(q[None], k[None], v[None], causal=True)[0]

    def run():
        h = model.w["embed"][tokens].float()
        for lw in model.w["layers"]:
            x = F.rms_norm(h, (d,), lw["attn_norm"], cfg.rms_eps).bfloat16()
            qkv = x @ lw["w_qkv"].T
            q = rope(qkv[:, : H * dh].view(n, H, dh))
            k = rope(qkv[:, H * dh: (H + Hkv) * dh].view(n, Hkv, dh))
            v = qkv[:, (H + Hkv) * dh:].view(n, Hkv, dh)
            o = attn(q, k, v).reshape(n, H * dh)
            h = h + (o @ lw["w_o"].T).float()
            x = F.rms_norm(h, (d,), lw["mlp_norm"], cfg.rms_eps).bfloat16()
            for i0 in range(0, n, 4096):  # (row blocks: the 70B full-recompute temporaries fit beside 140 GB of weights)
                gu = (x[i0:i0 + 4096] @ lw["w_gu"].T).view(-1, ff // 64, 2, 64)
                a = (F.silu(gu[:, :, 0].float()) * gu[:, :, 1].float()).bfloat16().reshape(-1, ff)
                h[i0:i0 + 4096] += (a @ lw["w_down"].T).float()
        last = F.rms_norm(h[-1:], (d,), model.w["final_norm"], cfg.rms_eps).bfloat16()
        return (last @ model.w["unembed_t"].T).argmax()

    for attn_name, attn in (("cudnn_sdpa", attn_cudnn), ("flash_attn", attn_flash)):
        try:
            run()
            break
        except Exception:  # backend unavailable on this box: try the next library
            continue
    return run, attn_name


def time_tiers(cc, model, req, steps, n_prompt):
    """f2: the same fix-up with every HIT chunk-cache in the pinned-host tier.
    Layer-wise preload (copy engine, L_p + 1 slot HBM ring, tiers.py) vs
    loading everything first (serial) vs all-HBM; device-timed."""
    import torch

    from paper_2502_15734_b200 import engine, tiers

    rate = tiers.calibrate_h2d(model)
    tp = tiers.TieredPool(model)
    segs = []
    for seg in req.segments:
        if seg.cache is None:
            segs.append(seg)
            continue
        c = seg.cache.copy()
        tp.move(c, tiers.HOST)
        segs.append(cc.Segment(tokens=seg.tokens, cache=c, recompute=seg.recompute,
                               recompute_depth=seg.recompute_depth))
    hreq = cc.build_request(segs, req.question)
    payloads = engine._payloads(model, hreq)
    dplan = engine.DevicePlan(model, hreq.token_ids, hreq.positions, hreq.is_pad, hreq.recompute_mask,
                              hreq.recompute_depth, hreq.segment_slots, payloads, hreq.question_span)
    ws = engine._workspace(model, dplan)
    ms, _ = time_device(model, dplan, ws, hreq, steps, 2, 1)
    depth = engine._HostPreload(model, dplan).depth
    torch.cuda.synchronize()
    host_bytes = sum(p.nbytes() for p, _ in dplan.host_payloads)
    # serial: copy all host slabs to HBM first, then the all-HBM step
    dst = torch.empty(host_bytes, dtype=torch.uint8, device=model.device)
    flat = [p.data.view(torch.uint8).reshape(-1) for p, _ in dplan.host_payloads]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    o = 0
    for f in flat:
        dst[o:o + f.numel()].copy_(f, non_blocking=True)
        o += f.numel()
    b.record()
    torch.cuda.synchronize()
    load_ms = a.elapsed_time(b)
    del ws, dst
    return {"workload": "config2 with all 10 HIT chunk-caches in pinned host memory",
            "layerwise_preload_ms": round(statistics.mean(ms), 3),
            "tokens_per_s": round(n_prompt / (statistics.mean(ms) / 1e3), 1),
            "preload_depth_Lp": depth, "host_bytes": int(host_bytes),
            "h2d_gbs_calibrated": round(rate / 1e9, 1),
            "serial_load_ms": round(load_ms, 3)}


def time_decode(cc, model, req, steps, peaks):
    """Greedy decode of `steps` tokens continuing the fix-up prefill
    (engine.DecodeSession: per-token GEMVs + split-KV attention, no host
    round trip), device-timed with CUDA events on the launching stream.
    Roofline: HBM — every token streams all weights once plus the KV of
    every layer (bf16)."""
    import torch

    from paper_2502_15734_b200 import engine

    res = cc.prefill(model, req, record_attention=False, stats=False)
    q1 = req.question_span[1] - 1
    h = torch.from_numpy(np.asarray(res.hidden[q1], np.float64).reshape(1, -1)).to(model.device, model.hidden_dtype)
    warm = engine.DecodeSession(model, res.kv, 4)
    warm.run(h)
    torch.cuda.synchronize()
    sess = engine.DecodeSession(model, res.kv, steps)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sess.run(h)
    b.record()
    torch.cuda.synchronize()
    if sess.replay_events is not None:  # steady state: graph replays of steps 1..n-1
        ms = sess.replay_events[0].elapsed_time(sess.replay_events[1]) * steps / (steps - 1)
    else:
        ms = a.elapsed_time(b)
    toks = sess.tokens[:steps].cpu().numpy().tolist()
    cfg = model.kcfg
    w_bytes = sum(t.numel() * t.element_size() for lw in model.w["layers"] for t in lw.values() if t is not None)
    w_bytes += model.w["unembed_t"].numel() * model.w["unembed_t"].element_size()
    n0 = res.kv.n_slots
    kv_bytes = sum(2 * (n0 + i + 1) * cfg.kv_width() * 2 * cfg.n_layers for i in range(steps)) / steps
    per_tok = (w_bytes + kv_bytes)
    ms_tok = ms / steps
    gbs = per_tok / (ms_tok / 1e3) / 1e9
    peak = peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 6536.4
    return {"tokens": steps, "tokens_per_s": round(steps / (ms / 1e3), 1), "ms_per_token": round(ms_tok, 4),
            "context_tokens": n0, "first_tokens": toks[:4],
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4),
                         "bytes_per_token": int(per_tok), "note": "all weights + the KV of every layer per token"}}


LLAMA3_8B_ORACLE = dict(n_heads=32, d_model=4096, d_head=128, vocab_size=128256, rpe_base=500000.0, n_kv_heads=8,
                        d_ff=14336, mlp="swiglu", norm_weight=True, rms_eps=1e-5)


def _use_all_cores():
    ncores = os.cpu_count() or 1
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = str(ncores)
    return ncores


def oracle_sample_seconds(weights, chunks, masks, question, caches) -> float:
    """Wall seconds of the oracle port (numpy float64) running
    len(weights["layers"]) full-width Llama-3-8B layers of the fix-up request
    (every slot, the given recompute rows, injected caches)."""
    from oracle import cachecraft_oracle as O

    ocfg = O.OracleConfig(n_layers=len(weights["layers"]), **LLAMA3_8B_ORACLE)
    lay = O.layout([{"tokens": t, "n_slots": t.size, "recompute": m} for t, m in zip(chunks, masks)], question)
    t0 = time.perf_counter()
    O.prefill(weights, ocfg, lay, caches, keep_weights=False)
    return time.perf_counter() - t0


def cpu_baseline(args, model, req):
    """Oracle port on the host cores, on a bounded sample of THE SAME request
    the GPU ran: the GPU model's own first `cpu_layers` layers (bf16 weights
    widened to float64), the stored variants' own cached K/V rows and the K9
    recompute rows, all 5152 slots; extrapolated to all layers.  Returns
    (tokens/s, cores, seconds, description)."""
    from oracle.from_device import cache_layers, weights_from_model

    ncores = _use_all_cores()
    nl = args.cpu_layers
    chunks = [np.asarray(seg.tokens) for seg in req.segments]
    w, remap = weights_from_model(model, chunks + [req.question], n_layers=nl)
    masks = [np.asarray(req.recompute_mask[s:e]) for s, e in req.segment_slots]
    caches = [cache_layers(seg.cache, nl) if seg.cache is not None else None for seg in req.segments]
    dt = oracle_sample_seconds(w, [remap(c) for c in chunks], masks, remap(req.question), caches)
    est = dt / nl * args.layers
    return req.n_tokens / est, ncores, dt, (
        f"oracle port (numpy fp64, {ncores} threads): {nl} of {args.layers} Llama-3-8B-shaped layers of the same "
        f"{req.n_slots}-slot fix-up request (the GPU model's weights and cached K/V, the K9 recompute rows) timed "
        f"({dt:.1f} s), extrapolated x{args.layers / nl:g}")


def reference_request(args):
    """The bench request rebuilt without the product package: the same seeded
    chunks and question as make_workload (rank 0), and the recompute rows the
    K9 top-k picks from the same seeded variant scores (oracle.select_tokens,
    planner.py:17-34)."""
    from oracle import cachecraft_oracle as O

    r = np.random.default_rng(1000)
    V = LLAMA3_8B_ORACLE["vocab_size"]
    chunks = [r.integers(0, V, args.chunk_len) for _ in range(args.chunks)]
    question = r.integers(0, V, args.question)
    rot = chunks[1:] + chunks[:1]  # creation order of make_workload
    scores = [r.standard_normal(c.size) for c in rot]
    scores = scores[-1:] + scores[:-1]  # back to request order
    masks = []
    for c, sc in zip(chunks, scores):
        m = np.zeros(c.size, bool)
        m[O.select_tokens(sc, args.ratio)] = True
        masks.append(m)
    return chunks, question, masks


def run_reference_arm(args, rank, world):
    """--impl reference: the reference algorithm on the host cores (the oracle
    port: the reference is pure numpy, no GPU code), same request, metric,
    unit and config as the product arm.  Each step times one full-width
    Llama-3-8B layer of the request (seeded float64 weights, seeded injected
    caches) and extrapolates to all layers."""
    if rank != 0:
        return
    ncores = _use_all_cores()
    chunks, question, masks = reference_request(args)
    g = np.random.default_rng(0)
    d, kvw, ff = 4096, 1024, 14336

    def nrm(rows, cols):
        return g.standard_normal((rows, cols), dtype=np.float32).astype(np.float64) / math.sqrt(rows)

    uniq = np.unique(np.concatenate(chunks + [question]))
    w = {"embed": g.standard_normal((uniq.size, d)), "final_norm": np.ones(d),
         "layers": [{"wq": nrm(d, d), "wk": nrm(d, kvw), "wv": nrm(d, kvw), "wo": nrm(d, d), "w_gate": nrm(d, ff),
                     "w_up": nrm(d, ff), "w_down": nrm(ff, d), "attn_norm": np.ones(d), "mlp_norm": np.ones(d)}]}
    caches = [([g.standard_normal((c.size, kvw))], [g.standard_normal((c.size, kvw))]) for c in chunks]
    remap = lambda t: np.searchsorted(uniq, t)  # noqa: E731
    n_prompt = sum(c.size for c in chunks) + question.size
    vals = []
    for i in range(args.warmup + args.steps):
        dt = oracle_sample_seconds(w, [remap(c) for c in chunks], masks, remap(question), caches)
        if i >= args.warmup:
            vals.append(n_prompt / (dt * args.layers))
    value = statistics.median(vals)
    desc = (f"oracle port (numpy fp64, {ncores} threads): 1 of {args.layers} Llama-3-8B-shaped layers of the same "
            f"{n_prompt}-token fix-up request per step (same chunks, question and K9 recompute rows; seeded "
            f"weights and caches), extrapolated x{args.layers}")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            # (extrapolated: one full request through all layers at the measured rate)
            "ms_per_step": round(n_prompt / value * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world),
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": ncores, "kind": "port", "sample": desc},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------


def _traffic(name, config):
    """DRAM bytes (read + write) per launch of `name` from the committed ncu
    capture of THIS config's step (profiles/traffic_<config>.json, written by
    tools/traffic_json.py from an ncu launch list); None if not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_{config}.json")) as fh:
            t = json.load(fh)
        return t["kernels"][name]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def roofline_obj(name, summ, peaks, bound, config="8b"):
    s = summ.get(name)
    if not s or s["ms_total"] <= 0:
        return None
    sec = s["ms_total"] / 1e3
    if bound == "tensor":
        ach = s["flops"] / sec / 1e12
        peak = peaks.get("bf16_tflops_sustained") or 1407.5
        return {"kernel": name, "bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 4), "traffic": _traffic(name, config), "launches": s["launches"],
                "avg_launch_us": round(s["ms_total"] * 1e3 / s["launches"], 2),
                "peak_source": "measured sustained (MEASURED_PEAKS.json)"}
    ach = s["bytes"] / sec / 1e9
    peak = peaks.get("hbm_gbs") or 6536.4
    return {"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4), "traffic": _traffic(name, config), "launches": s["launches"],
            "algorithmic_bytes_per_launch": int(s["bytes"] / s["launches"]),
            "avg_launch_us": round(s["ms_total"] * 1e3 / s["launches"], 2),
            "peak_source": "measured copy bandwidth (MEASURED_PEAKS.json)"}


def run_zipf(args, rank, world):
    """Config 3: Llama-3-8B shapes, a Zipf trace of 10x512-token retrievals
    (top 5% of chunks take ~60% of retrievals, harness.py:125-144) replayed
    request by request through the public API (build_plan -> prefill with
    creation statistics for misses -> store update), requests sharded across
    ranks by chunk affinity, 15% recompute per hit.  Wall-clock (end-to-end)
    prompt tokens/s over the steady state (first 20 requests of each rank are
    warm-up), summed over ranks; p50/p99 TTFT; same trace under full
    recompute and exact-prefix caching."""
    import torch

    import paper_2502_15734_b200 as cc
    from paper_2502_15734_b200 import harness, parallel

    cfg = cc.ModelConfig.llama3_8b(n_layers=args.layers, dtype="bf16", seed=0)
    model = cc.build_model(cfg)
    n_chunks, k = 200, args.chunks
    n_req = args.requests * world
    gen = dict(chunk_len_range=(args.chunk_len, args.chunk_len), question_len_range=(args.question, args.question),
               vocab_size=cfg.vocab_size)
    skew = harness.fit_zipf_skew(n_chunks, k, n_req, target_share=0.6, seed=3, iterations=12, **gen)
    trace = harness.gen_synthetic(n_chunks, skew, k, n_req, seed=3, **gen)
    mine = parallel.shard_requests(trace.records, rank, world, "affinity")
    warm = min(20, max(0, len(mine) - 5))
    out = {}
    for policy in ("cachecraft", "exact_prefix", "full_recompute"):
        store = cc.VariantStore(cc.StoreConfig(max_chunks=100, variants_per_chunk=5))
        barrier(world)
        rep = harness.replay_gpu(trace, model, store, policy=policy, warmup=warm, cfo_override=args.ratio,
                                measure_deviation=False, records=mine)
        agg = rep.aggregate()
        steady = rep.steady_state()
        tok = float(sum(r.tokens_total for r in steady))
        wall = sum(r.ttft for r in steady)
        wall_max = allreduce_max(wall, world)
        tok_all = tok
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([tok], dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            tok_all = float(t.item())
        out[policy] = {"tokens_per_s": tok_all / wall_max if wall_max else 0.0, "ttft_p50_ms": agg.get("ttft_p50_ms"),
                       "ttft_p99_ms": agg.get("ttft_p99_ms"), "hit_rate": agg.get("hit_rate"),
                       "recompute_fraction": agg.get("recompute_fraction"), "requests": agg.get("n_requests")}
        del store
        torch.cuda.empty_cache()
    if rank != 0:
        return
    cc_ = out["cachecraft"]
    line = {
        "metric": "prefill tokens/sec on a Zipf chunk-reuse trace at 15% recompute per hit (Llama-3-8B shapes)",
        "value": round(cc_["tokens_per_s"], 1), "unit": UNIT, "n_gpus": world, "steps": cc_["requests"],
        "warmup": warm, "ms_per_step": round(cc_["ttft_p50_ms"], 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic Zipf trace (random tokens, random-init weights)",
        "config": {"workload": f"config3: {n_req} requests x {k} chunks of {args.chunk_len} tokens + "
                               f"{args.question}-token question from a {n_chunks}-chunk corpus, zipf s={skew:.3f} "
                               f"(top-5% share {harness.top_share(trace):.2f}), store N=100 M=5 per GPU, "
                               "affinity request sharding", "parallelism": f"request-sharded x{world}"},
        "e2e": {"value": round(cc_["tokens_per_s"], 1), "unit": UNIT, "path": "replay_gpu (public API per request)"},
        "policies": out,
        "speedup_vs_full_recompute": round(cc_["tokens_per_s"] / out["full_recompute"]["tokens_per_s"], 3),
        "speedup_vs_exact_prefix": round(cc_["tokens_per_s"] / out["exact_prefix"]["tokens_per_s"], 3),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        # host-only arm: rank 0 runs, other ranks exit without work
        run_reference_arm(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, world = dist_init(args)
    if args.config == "zipf":
        run_zipf(args, rank, world)
        return
    import torch

    from paper_2502_15734_b200 import _native
    from paper_2502_15734_b200 import engine as engine_mod

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

    cc, model, store, chunks, question = make_workload(args, rank)
    model.l2_prefetch = os.environ.get("CCB_L2PF") == "1"  # side-stream weight prefetch: measured neutral, off
    plan, req, dplan, ws = resident_plan(cc, model, store, chunks, question, args.ratio)
    n_prompt = req.n_tokens
    n_recomputed = plan.tokens_recomputed()

    # ---- value: device-timed fix-up -----------------------------------------
    # (a) one request at a time (latency; per-kernel CUDA events on the last
    # timed step only: an event pair around every launch family costs ~0.8 ms
    # over a whole step, one step still gives every family its 32 launches)
    # (b) serving throughput: K requests in flight on K CUDA streams, each
    # replaying its own resident request (distinct questions); the value
    K = args.streams if args.streams > 0 else {"8b": 6, "8b-32k": 2, "70b": 1}[args.config]
    calls0 = sum(_native.calls.values())
    barrier(world)
    tp_mode = args.config == "70b" and world > 1
    with Clocks(torch.cuda.current_device()) as clk:
        n_timed = 1
        ms, timer = time_device(model, dplan, ws, req, args.steps, args.warmup, world, timer_steps=n_timed)
        launches = (sum(_native.calls.values()) - calls0) // (args.steps + args.warmup)
        ms_step = statistics.mean(ms)
        ms_max = allreduce_max(ms_step, world)
        value_single = n_prompt * (1 if tp_mode else world) / (ms_max / 1e3)
        ms_req = ms_max
        if K > 1:
            vq = np.random.default_rng(4242 + rank)
            runs = []
            for _ in range(K):
                _, rq_k, dp_k, ws_k = resident_plan(cc, model, store, chunks,
                                                    vq.integers(0, model.config.vocab_size, args.question), args.ratio)
                runs.append((dp_k, ws_k, rq_k))
            ms_req = allreduce_max(time_device_streams(model, runs, args.steps, args.warmup, world), world)
            del runs
    clocks = clk.summary()
    value = n_prompt * (1 if tp_mode else world) / (ms_req / 1e3)
    summ = timer.summary()

    # ---- e2e: public API with host buffers ----------------------------------
    # every request carries its own question (same chunks, same length), so no
    # two requests of the stream are identical
    qr = np.random.default_rng(77 + rank)
    questions = [qr.integers(0, model.config.vocab_size, args.question) for _ in range(2 * (args.warmup + args.steps) + 2)]
    # (a) TTFT: one request at a time, planning included, first token on host
    e2e_ms, ttft = [], []
    h2d = d2h = 0
    for i in range(args.warmup + args.steps):
        barrier(world)
        t0 = time.perf_counter()
        p = cc.build_plan(chunks, questions[i], store, alpha=1.0, cfo_override=args.ratio)
        rq = cc.plan_to_request(p)
        res = cc.prefill(model, rq, record_attention=False, stats=False, first_token=True)
        tok = res.first_token
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_ms.append((t1 - t0) * 1e3)
            h2d = res.extras["plan"].h2d_bytes + sum(8 * len(np.asarray(cp.recompute)) + 64 for cp in p.chunks)
            d2h = 4 + sum(4 * len(cp.recompute) for cp in p.chunks if cp.recompute is not None)
        del res
    ttft_p50 = statistics.median(e2e_ms)
    # (b) throughput: a request stream through the same API, pipelined the way
    # a server runs it — request i+1 is planned (host scoring, K9 on the
    # planning stream, layout, H2D) while request i computes; every request's
    # copies and its first-token readback stay inside the timed region
    # Two requests in flight: request i is enqueued before request i-1's first
    # token is read back (an event behind i-1's kernels, not a stream sync),
    # so the GPU runs the requests back to back
    # K requests in flight, request i on stream i % K (the serving mode of
    # (b) above): each request is planned and enqueued, and the oldest one's
    # first token is read back once K are in flight
    barrier(world)
    t_start = time.perf_counter()
    qs = questions[args.warmup + args.steps:]
    e2e_streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(K - 1)]
    done = []
    inflight = []
    n_req = args.warmup + args.steps + K
    with engine_mod.concurrent_streams() if K > 1 else contextlib.nullcontext():
        for i in range(n_req):
            with torch.cuda.stream(e2e_streams[i % K]):
                p = cc.build_plan(chunks, qs[i % len(qs)], store, alpha=1.0, cfo_override=args.ratio)
                inflight.append(cc.prefill(model, cc.plan_to_request(p), record_attention=False, stats=False,
                                           first_token=True))
            if len(inflight) > K - 1 and len(done) < args.warmup + args.steps:
                tok = inflight.pop(0).first_token
                done.append(time.perf_counter())
        for r_ in inflight:
            tok = r_.first_token
        torch.cuda.synchronize()
        del inflight
    per_req = (done[-1] - done[args.warmup - 1]) / args.steps if args.warmup > 0 else (done[-1] - t_start) / args.steps
    e2e_mean = allreduce_max(per_req * 1e3, world)
    e2e_value = n_prompt * (1 if tp_mode else world) / (e2e_mean / 1e3)

    # ---- decode continuation on the repaired KV (f3) ------------------------
    decode = None
    if args.decode_steps > 0 and not tp_mode:
        torch.cuda.empty_cache()
        try:
            decode = time_decode(cc, model, req, args.decode_steps, peaks)
        except torch.cuda.OutOfMemoryError as e:  # 70B on one GPU: weights leave ~2 GB free
            decode = {"skipped": "out of memory for the decode KV capacity buffers: " + str(e).splitlines()[0][:120]}
        torch.cuda.empty_cache()

    tiers_leg = None
    if args.tiers and not tp_mode:
        try:
            tiers_leg = time_tiers(cc, model, req, max(3, args.steps // 2), n_prompt)
        except torch.cuda.OutOfMemoryError as e:
            tiers_leg = {"skipped": "out of memory: " + str(e).splitlines()[0][:120]}
        torch.cuda.empty_cache()
    if tiers_leg is not None and "skipped" not in tiers_leg:
        tiers_leg["all_hbm_ms"] = round(ms_step, 3)
        tiers_leg["serial_ms"] = round(tiers_leg["serial_load_ms"] + ms_step, 3)

    # ---- baselines on the same GPU --------------------------------------------
    baselines = {}
    if not args.no_baselines:
        reqf, dpf, wsf = full_plan(cc, model, chunks, question)
        msf, tf = time_device(model, dpf, wsf, reqf, max(3, args.steps // 2), 2, world, timer_steps=1)
        del wsf
        baselines["full_recompute_ours"] = {"tokens_per_s": round(n_prompt / (statistics.mean(msf) / 1e3), 1),
                                            "ms_per_step": round(statistics.mean(msf), 3),
                                            "rows_computed": n_prompt}
        reqp, dpp, wsp = prefix_plan(cc, model, store, chunks, question, int(round(0.6 * len(chunks))))
        msp, _ = time_device(model, dpp, wsp, reqp, max(3, args.steps // 2), 2, world)
        del wsp
        baselines["prefix_cache_60pct_ours"] = {"tokens_per_s": round(n_prompt / (statistics.mean(msp) / 1e3), 1),
                                                "ms_per_step": round(statistics.mean(msp), 3)}
        if K > 1:  # full recompute at the same concurrency as the value
            fq = np.random.default_rng(999)
            runs_f = []
            for _ in range(K):
                rq_f, dp_f, ws_f = full_plan(cc, model, chunks, fq.integers(0, model.config.vocab_size, args.question))
                runs_f.append((dp_f, ws_f, rq_f))
            msf_k = allreduce_max(time_device_streams(model, runs_f, max(3, args.steps // 2), 2, world), world)
            del runs_f
            baselines["full_recompute_ours_streams"] = {"tokens_per_s": round(n_prompt / (msf_k / 1e3), 1),
                                                        "ms_per_request": round(msf_k, 3), "requests_in_flight": K}
            baselines["speedup_vs_full_recompute_ours_same_concurrency"] = round(msf_k / ms_req, 3)
        # the same three policies through the public API, one request at a
        # time with host token lists: p50 TTFT (submit -> first token on host)
        n_hit = int(round(0.6 * len(chunks)))

        def fixup_req(i):
            return cc.plan_to_request(cc.build_plan(chunks, questions[i], store, alpha=1.0, cfo_override=args.ratio))

        def full_req(i):
            return cc.plain_request(*chunks, questions[i])

        def prefix_req(i):
            segs = [cc.Segment(tokens=c, cache=store.lookup(cc.chunk_hash(c))[0].cache) if j < n_hit
                    else cc.Segment(tokens=c) for j, c in enumerate(chunks)]
            return cc.build_request(segs, questions[i])

        api = {}
        for name, mk in (("fix_up_15pct", fixup_req), ("full_recompute", full_req), ("prefix_cache_60pct", prefix_req)):
            ts = []
            for i in range(args.warmup + max(3, args.steps // 2)):
                barrier(world)
                t0 = time.perf_counter()
                res = cc.prefill(model, mk(i), record_attention=False, stats=False, first_token=True)
                _ = res.first_token
                if i >= args.warmup:
                    ts.append((time.perf_counter() - t0) * 1e3)
                del res
            api[name] = {"ttft_p50_ms": round(statistics.median(ts), 3),
                         "tokens_per_s": round(n_prompt / (statistics.median(ts) / 1e3), 1)}
        api["speedup_ttft_vs_full_recompute"] = round(api["full_recompute"]["ttft_p50_ms"]
                                                      / api["fix_up_15pct"]["ttft_p50_ms"], 3)
        api["speedup_ttft_vs_prefix_cache"] = round(api["prefix_cache_60pct"]["ttft_p50_ms"]
                                                    / api["fix_up_15pct"]["ttft_p50_ms"], 3)
        baselines["public_api_ttft"] = api
        # K8 on the MISS path (harness.py:331-354): a store miss prefills its
        # chunks fresh WITH creation statistics (cc_segment_mass: per-row mass
        # per key segment, recomputed from q / lse; cc_chunk_stats) so the new
        # variants can be scored.  Same 10 x 512 + 32 request, all chunks new.
        miss = {}
        for name, st in (("no_stats", False), ("with_creation_stats", True)):
            ts = []
            for i in range(args.warmup + 3):
                barrier(world)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = cc.prefill(model, full_req(i), record_attention=False, stats=st)
                if st:
                    cc.creation_stats(res, list(range(len(chunks) + 1)), list(range(len(chunks))))
                torch.cuda.synchronize()
                if i >= args.warmup:
                    ts.append((time.perf_counter() - t0) * 1e3)
                del res
            miss[name + "_ms"] = round(statistics.median(ts), 3)
        miss["k8_cost_ms"] = round(miss["with_creation_stats_ms"] - miss["no_stats_ms"], 3)
        miss["k8_share"] = round(miss["k8_cost_ms"] / miss["with_creation_stats_ms"], 4)
        # K8's own launches, device-timed on the launching stream (same MISS
        # request, every chunk span + the question as stats segments)
        from paper_2502_15734_b200 import engine as E_

        reqm, dpm, wsm = full_plan(cc, model, chunks, question)
        segm = list(reqm.segment_slots) + [tuple(reqm.question_span)]
        dpm.stats_segments = segm
        E_._attach_stats_rows(model, dpm, segm)
        tk8 = E_.KernelTimer()
        for i in range(args.warmup + 2):
            E_.execute(model, dpm, wsm, stats=True, timer=tk8 if i >= args.warmup else None)
        torch.cuda.synchronize()
        miss["segment_mass_roofline"] = roofline_obj("segment_mass", tk8.summary(), peaks, "tensor", args.config)
        del wsm
        baselines["miss_path_full_prefill"] = miss
    if not args.no_baselines and not tp_mode:
        toks = torch.from_numpy(np.concatenate(chunks + [question]).astype(np.int64)).cuda()
        run, attn_name = torch_reference_full(model, toks)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        ev = []
        for _ in range(max(3, args.steps // 2)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        mst = statistics.mean(a.elapsed_time(b) for a, b in ev)
        baselines["full_recompute_cublas_" + attn_name] = {"tokens_per_s": round(n_prompt / (mst / 1e3), 1),
                                                          "ms_per_step": round(mst, 3)}
        baselines["speedup_vs_full_recompute_ours"] = round(baselines["full_recompute_ours"]["ms_per_step"] / ms_step, 3)
        baselines["speedup_vs_full_recompute_cublas"] = round(mst / ms_step, 3)

    sweep = None
    if args.sweep:
        sweep = {}
        for r in (0.0, 0.05, 0.10, 0.15, 0.20, 0.30, 0.40, 0.50):
            _, rq_, dp_, ws_ = resident_plan(cc, model, store, chunks, question, r)
            m_, _ = time_device(model, dp_, ws_, rq_, 5, 2, world)
            sweep[f"{r:.2f}"] = {"ms": round(statistics.mean(m_), 3),
                                 "tokens_per_s": round(n_prompt / (statistics.mean(m_) / 1e3), 1)}
            del ws_

    cpu = None
    if rank == 0 and not args.no_cpu and args.config == "8b":
        v, cores, dt, desc = cpu_baseline(args, model, req)
        cpu = {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "port", "sample": desc}

    if rank != 0:
        return
    from paper_2502_15734_b200 import _native as N_

    wcfg = workload_config(args, world)
    assert (wcfg["prompt_tokens"], wcfg["recomputed_rows"]) == (n_prompt, n_recomputed), (wcfg, n_prompt, n_recomputed)
    N_.assert_tensor_core_only()  # every bf16 GEMM / attention of the run ran on tcgen05
    gemm_roof = roofline_obj("gemm", summ, peaks, "tensor", args.config)
    kernels = [k for k in (roofline_obj("gather_rope", summ, peaks, "hbm", args.config),
                           roofline_obj("attention", summ, peaks, "tensor", args.config),
                           roofline_obj("rmsnorm", summ, peaks, "hbm", args.config),
                           roofline_obj("rope_scatter", summ, peaks, "hbm", args.config)) if k]
    share = {k: round(v["ms_total"] / (sum(ms[-n_timed:]) or 1), 4) for k, v in summ.items()}
    line = {
        "metric": METRIC if args.config == "8b" else METRIC.replace("Llama-3-8B shapes, 10x512+32", {
            "8b-32k": "Llama-3-8B shapes, 64x512+32", "70b": "Llama-3-70B shapes, 16x1024+32"}[args.config]),
        "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_req, 4), "higher_is_better": True,
        "scaling": "strong" if tp_mode else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, random token chunks)",
        "config": wcfg,
        "ttft_ms": {"p50_e2e": round(ttft_p50, 3), "device_mean": round(ms_step, 3)},
        "requests_in_flight": K,
        "single_request": {"value": round(value_single, 1), "unit": UNIT, "ms_per_request": round(ms_max, 4),
                           "note": "one request at a time on one stream (device-timed)"},
        "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "path": "build_plan -> plan_to_request -> prefill(first_token=True)",
                "mode": f"request stream with {K} requests in flight on {K} CUDA streams (a request's first token "
                        "is read back once the next ones are enqueued; planning overlapped with compute); "
                        "serial TTFT in ttft_ms.p50_e2e"},
        "roofline": gemm_roof,
        "roofline_kernels": kernels,
        "kernel_time_share": share,
        "gpu_launches": int(launches),
        "bf16_simt_launches": N_.bf16_simt_launches(),
        "cpu_baseline": cpu,
        "baselines": baselines,
        "clocks": clocks,
    }
    if sweep:
        line["recompute_sweep"] = sweep
    if decode:
        line["decode"] = decode
    if tiers_leg:
        line["tiers"] = tiers_leg
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
