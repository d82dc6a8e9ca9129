"""Trace synthesis and GPU replay of the chunk-cache pipeline (
cachecraft/harness.py:67-144, :324-591).

``replay_gpu`` drives the hot path request by request exactly like the
reference's ``replay``: plan (host decisions + K9 selection on the GPU) ->
partial prefill (device engine, K8 statistics when a chunk misses) ->
optional focused-chunk early termination (Algorithm 1 on the device's
question->chunk masses, then the reference's second pass) -> store update
(new variants from MISS chunks via K10 extraction, f_r touch for HITs).  The
baseline policies run for real on the GPU: ``full_recompute`` (plain
prefill), ``full_cache_naive`` (latest variant, nothing recomputed) and
``exact_prefix`` (prefix caching: the longest chunk-boundary prefix seen
before is reused verbatim from an HBM prefix registry, the rest computed).
The tier simulator (simulated TTFT) is out of scope; TTFT here is measured.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import time
from collections import OrderedDict
from dataclasses import asdict, dataclass, field

import numpy as np

from .errors import ArgumentError, IoError
from .model import Segment, build_request, extract_chunk_cache, plain_request, prefill
from .planner import HIT, MISS, ChunkPlan, InferencePlan, apply_early_termination, build_plan, plan_to_request, \
    predict_focused
from .scoring import cci
from .stats import creation_stats, question_stream
from .store import chunk_hash
from .tiers import place_and_migrate

POLICIES = ("cachecraft", "full_recompute", "full_cache_naive", "exact_prefix")
DEFAULT_WARMUP = 20  # requests excluded from aggregates (harness.py:47)
DEFAULT_QUEUE_WAIT = 0.32  # the reference's typical queue wait, seconds (tiers.py:24)


@dataclass
class TraceRecord:
    request_id: int
    chunk_ids: list
    question: np.ndarray
    arrival_s: float


@dataclass
class Trace:
    records: list
    corpus: dict

    def __len__(self) -> int:
        return len(self.records)


def gen_synthetic(n_chunks: int, zipf_s: float, k: int, n_requests: int, chunk_len_range=(16, 64), seed: int = 0,
                  question_len_range=(8, 16), vocab_size: int = 256, arrival_rate: float = 2.0) -> Trace:
    """Zipf-popularity trace, same draw order as harness.py:84-106 (so a seed
    gives the reference's trace): corpus lengths/tokens, then per request k
    distinct chunks, a question and an exponential inter-arrival gap."""
    if k > n_chunks:
        raise ArgumentError(f"k ({k}) cannot exceed the corpus size ({n_chunks})")
    if n_chunks < 1 or n_requests < 0:
        raise ArgumentError("corpus and request counts must be non-negative")
    g = np.random.default_rng(seed)
    lo, hi = chunk_len_range
    corpus = {}
    for cid in range(n_chunks):
        length = int(g.integers(lo, hi + 1))
        corpus[cid] = g.integers(0, vocab_size, size=length)
    pop = (1.0 / np.arange(1, n_chunks + 1)) ** zipf_s
    pop /= pop.sum()
    qlo, qhi = question_len_range
    t = 0.0
    recs = []
    for rid in range(n_requests):
        pick = g.choice(n_chunks, size=k, replace=False, p=pop)
        q = g.integers(0, vocab_size, size=int(g.integers(qlo, qhi + 1)))
        t += float(g.exponential(1.0 / arrival_rate))
        recs.append(TraceRecord(request_id=rid, chunk_ids=[int(c) for c in pick], question=q, arrival_s=t))
    return Trace(records=recs, corpus=corpus)


def top_share(trace: Trace, top_fraction: float = 0.05) -> float:
    """Fraction of retrievals landing on the most popular chunks (harness.py:110-122)."""
    counts: dict = {}
    for rec in trace.records:
        for cid in rec.chunk_ids:
            counts[cid] = counts.get(cid, 0) + 1
    total = sum(counts.values())
    if total == 0:
        return 0.0
    n_top = max(1, int(math.ceil(top_fraction * len(trace.corpus))))
    return sum(sorted(counts.values(), reverse=True)[:n_top]) / total


def fit_zipf_skew(n_chunks: int, k: int, n_requests: int, target_share: float = 0.6, seed: int = 0,
                  iterations: int = 18, **gen_kwargs) -> float:
    """Bisect the Zipf exponent in [0, 4] until the top-5% share meets the
    target (harness.py:125-144)."""
    lo, hi = 0.0, 4.0
    for _ in range(iterations):
        mid = (lo + hi) / 2
        if top_share(gen_synthetic(n_chunks, mid, k, n_requests, seed=seed, **gen_kwargs)) < target_share:
            lo = mid
        else:
            hi = mid
    return (lo + hi) / 2


def save_trace(trace: Trace, path):
    """JSON lines, one request per line ({id, chunks, question, arrival_s});
    the chunk contents go to ``<path>.corpus.json`` (harness.py:150-171)."""
    try:
        with open(path, "w", encoding="utf-8") as fh:
            fh.writelines(json.dumps({"id": r.request_id, "chunks": list(r.chunk_ids),
                                      "question": np.asarray(r.question).astype(int).tolist(),
                                      "arrival_s": r.arrival_s}) + "\n" for r in trace.records)
        with open(_corpus_path(path), "w", encoding="utf-8") as fh:
            json.dump({str(c): np.asarray(t).astype(int).tolist() for c, t in trace.corpus.items()}, fh)
    except OSError as exc:
        raise IoError(f"cannot write trace {path}: {exc}") from exc


def load_trace(path) -> Trace:
    """Inverse of save_trace (harness.py:174-199); integer-looking corpus keys
    come back as ints."""
    try:
        with open(path, encoding="utf-8") as fh:
            objs = [json.loads(line) for line in fh if line.strip()]
        with open(_corpus_path(path), encoding="utf-8") as fh:
            raw = json.load(fh)
    except OSError as exc:
        raise IoError(f"cannot read trace {path}: {exc}") from exc
    records = [TraceRecord(request_id=o["id"], chunk_ids=o["chunks"], question=np.asarray(o["question"], np.int64),
                           arrival_s=o["arrival_s"]) for o in objs]
    corpus = {(int(k) if k.lstrip("-").isdigit() else k): np.asarray(v, dtype=np.int64) for k, v in raw.items()}
    return Trace(records=records, corpus=corpus)


def _corpus_path(path) -> str:
    return os.fspath(path) + ".corpus.json"


@dataclass
class RequestMetrics:
    """Per-request accounting (harness.py:206-221).  ``ttft`` is the MEASURED
    time to first token in seconds (submit -> greedy token on the host), not
    the reference's tier-simulator estimate; ``first_token`` is the token."""

    request_id: int
    arrival_s: float
    k: int
    hits: int
    tokens_total: int
    tokens_computed: int
    tokens_reused: int
    recompute_fraction: float
    tokens_hit_total: int
    tokens_hit_recomputed: int
    token_layers: int
    deviation: float
    ttft: float
    mean_cfo: float
    first_token: int | None = None


@dataclass
class Report:
    """One policy's replay (harness.py:224-262); ``aggregate`` adds the
    measured throughput and TTFT percentiles to the reference's keys."""

    policy: str
    alpha: float
    warmup: int
    requests: list = field(default_factory=list)

    def steady_state(self) -> list:
        return self.requests[self.warmup:]

    def aggregate(self) -> dict:
        rows = self.steady_state()
        keys = ("n_requests", "tokens_total", "tokens_computed", "tokens_reused", "recompute_fraction",
                "hit_recompute_fraction", "mean_deviation", "mean_ttft", "hit_rate", "mean_cfo", "token_layers")
        if not rows:
            return {k: (0 if k in ("n_requests", "tokens_total", "tokens_computed", "tokens_reused", "token_layers")
                        else 0.0) for k in keys}
        total = sum(r.tokens_total for r in rows)
        computed = sum(r.tokens_computed for r in rows)
        hit_total = sum(r.tokens_hit_total for r in rows)
        ttft = np.array([r.ttft for r in rows])
        out = dict(zip(keys, (
            len(rows), total, computed, total - computed, computed / total if total else 0.0,
            sum(r.tokens_hit_recomputed for r in rows) / hit_total if hit_total else 0.0,
            float(np.mean([r.deviation for r in rows])), float(ttft.mean()),
            sum(r.hits for r in rows) / max(1, sum(r.k for r in rows)),
            float(np.mean([r.mean_cfo for r in rows])), sum(r.token_layers for r in rows))))
        out["prompt_tokens_per_s"] = total / ttft.sum() if ttft.sum() > 0 else 0.0
        out["ttft_p50_ms"] = float(np.median(ttft) * 1e3)
        out["ttft_p99_ms"] = float(np.percentile(ttft, 99) * 1e3)
        return out


_CSV_COLUMNS = ("request_id", "arrival_s", "k", "hits", "tokens_total", "tokens_computed", "tokens_reused",
                "recompute_fraction", "tokens_hit_total", "tokens_hit_recomputed", "token_layers", "deviation",
                "ttft", "mean_cfo")


def export_report(report: Report, path, fmt: str = "csv"):
    """CSV: the steady-state rows, floats at 6 significant digits; JSON: the
    whole report plus its aggregate, exact round trip (harness.py:283-318)."""
    if fmt not in ("csv", "json"):
        raise ArgumentError(f"unknown export format {fmt!r}")
    try:
        with open(path, "w", encoding="utf-8") as fh:
            if fmt == "json":
                json.dump({"policy": report.policy, "alpha": report.alpha, "warmup": report.warmup,
                           "aggregate": report.aggregate(), "requests": [asdict(r) for r in report.requests]},
                          fh, indent=2)
                return
            fh.write(",".join(_CSV_COLUMNS) + "\n")
            for r in report.steady_state():
                cells = (getattr(r, c) for c in _CSV_COLUMNS)
                fh.write(",".join(f"{v:.6g}" if isinstance(v, float) else str(v) for v in cells) + "\n")
    except OSError as exc:
        raise IoError(f"cannot write report {path}: {exc}") from exc


def load_report(path) -> Report:
    try:
        with open(path, encoding="utf-8") as fh:
            obj = json.load(fh)
    except OSError as exc:
        raise IoError(f"cannot read report {path}: {exc}") from exc
    return Report(policy=obj["policy"], alpha=obj["alpha"], warmup=obj["warmup"],
                  requests=[RequestMetrics(**r) for r in obj["requests"]])


def question_deviation(hidden_rows, oracle_rows) -> float:
    """Mean per-token L2 distance over the question span (harness.py:364-370)."""
    hidden_rows, oracle_rows = np.asarray(hidden_rows), np.asarray(oracle_rows)
    if hidden_rows.shape != oracle_rows.shape:
        raise ArgumentError("question spans differ between run and oracle")
    if hidden_rows.shape[0] == 0:
        return 0.0
    return float(np.linalg.norm(hidden_rows - oracle_rows, axis=1).mean())


_deviation = question_deviation


def _naive_plan(chunk_tokens, hashes, question, store, alpha) -> InferencePlan:
    """Latest variant of every cached chunk, nothing recomputed (harness.py:373-396)."""
    out = []
    for toks, cid in zip(chunk_tokens, hashes):
        vs = store.lookup(cid)
        if vs:
            v = max(vs, key=lambda x: (x.created_at, x.variant_id))
            out.append(ChunkPlan(chunk_id=cid, status=HIT, tokens=toks, n_tokens=toks.size, n_slots=v.cache.n_slots,
                                 variant_id=v.variant_id, cfo=0.0, recompute=np.empty(0, dtype=np.int64),
                                 cache=v.cache))
        else:
            out.append(ChunkPlan(chunk_id=cid, status=MISS, tokens=toks, n_tokens=toks.size, n_slots=toks.size))
    return InferencePlan(chunks=out, question=question, alpha=alpha)


def _execute_planned(model, plan, hashes, store, use_focus, first_token, two_pass=False):
    """harness.py:399-451 on the device engine.  Early termination runs online
    in the single prefill (engine.OnlineFocus) unless ``two_pass`` asks for the
    reference's run-predict-rerun sequence."""
    n_layers = model.config.n_layers
    has_miss = any(cp.status == MISS for cp in plan.chunks)
    can_terminate = use_focus and len(plan.chunks) >= 3 and any(
        cp.status == HIT and cp.recompute is not None and cp.recompute.size for cp in plan.chunks)
    request = plan_to_request(plan)
    if can_terminate and not two_pass:
        result = prefill(model, request, stats=True, record_attention=False, first_token=first_token,
                         focus_window=plan.focus_window)
        if result.extras.get("focus_cut"):
            plan = apply_early_termination(plan, result.extras["focus"])
    else:
        result = prefill(model, request, stats=has_miss or can_terminate, record_attention=False,
                         first_token=first_token)
        if can_terminate:
            focus = predict_focused(question_stream(result), plan.focus_window)
            unfocused = set(range(len(plan.chunks))) - set(focus.focused)
            rerun = focus.cutoff_layer < n_layers and any(
                plan.chunks[i].status == HIT and plan.chunks[i].recompute is not None
                and plan.chunks[i].recompute.size for i in unfocused)
            if rerun:
                plan = apply_early_termination(plan, focus)
                request = plan_to_request(plan)
                result = prefill(model, request, stats=has_miss, record_attention=False, first_token=first_token)
    miss_idx = [i for i, cp in enumerate(plan.chunks) if cp.status == MISS]
    stats = creation_stats(result, hashes, miss_idx) if miss_idx else {}
    for i, cp in enumerate(plan.chunks):
        if cp.status == MISS:
            prefix, a_bar, b_bar, scores = stats[i]
            s0, s1 = request.segment_slots[i]
            cache = extract_chunk_cache(result, s0, s1, source_prefix=prefix.chunk_ids)
            store.insert(cp.chunk_id, prefix=prefix, a_bar=a_bar, b_bar=b_bar, cci=cci(a_bar, b_bar),
                         token_scores=scores, cache=cache)
        else:
            store.touch(cp.variant_id, cp.cfo)
    return result, plan, request


def _prefix_keys(chunk_tokens):
    """Running content hashes of every chunk-boundary prefix (harness.py:454-461)."""
    h = hashlib.blake2b(digest_size=16)
    keys = []
    for toks in chunk_tokens:
        h.update(np.asarray(toks, dtype=np.int64).tobytes())
        keys.append(h.copy().hexdigest())
    return keys


class PrefixRegistry:
    """GPU prefix cache for the exact_prefix baseline: prefix key -> the
    chunk cache computed in exactly that prefix context (LRU-bounded)."""

    def __init__(self, capacity: int = 512):
        self.capacity = capacity
        self._m: OrderedDict = OrderedDict()

    def get(self, key):
        c = self._m.get(key)
        if c is not None:
            self._m.move_to_end(key)
        return c

    def put(self, key, cache):
        self._m[key] = cache
        self._m.move_to_end(key)
        while len(self._m) > self.capacity:
            self._m.popitem(last=False)


def replay_gpu(trace: Trace, model, store=None, alpha: float = 1.0, policy: str = "cachecraft", warmup: int = 20,
               focus_window: int = 3, use_focus: bool = True, cfo_override: float | None = None,
               measure_deviation: bool = True, first_token: bool = True, registry: PrefixRegistry | None = None,
               records=None, two_pass: bool = False, tier_pool=None, tier_cfg=None) -> Report:
    """Replay (a shard of) a trace under one policy on the GPU.  ``records``
    restricts the run to this rank's requests (``parallel.shard_requests``)."""
    import torch

    if policy not in POLICIES:
        raise ArgumentError(f"unknown policy {policy!r}; expected one of {POLICIES}")
    L = model.config.n_layers
    report = Report(policy=policy, alpha=alpha, warmup=warmup)
    if store is not None:
        # size the HBM pool for the store's N*M variants up front (growth copies the pool)
        longest = max(len(t) for t in trace.corpus.values())
        need = (store.config.capacity + 64) * -(-longest // 16)
        if model.pool.n_blocks < need:
            model.pool.reserve(need)
    registry = registry if registry is not None else PrefixRegistry()
    for rec in (trace.records if records is None else records):
        chunk_tokens = [np.asarray(trace.corpus[c], dtype=np.int64) for c in rec.chunk_ids]
        question = np.asarray(rec.question, dtype=np.int64)
        k = len(chunk_tokens)
        total = sum(t.size for t in chunk_tokens) + question.size
        hashes = [chunk_hash(t) for t in chunk_tokens]
        oracle_q = None
        if measure_deviation and policy != "full_recompute":
            full = prefill(model, build_request([Segment(tokens=t) for t in chunk_tokens], question), stats=False,
                           record_attention=False)
            oracle_q = full.hidden[slice(*full.question_span)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tok = None
        if policy == "full_recompute":
            res = prefill(model, plain_request(*chunk_tokens, question), stats=False, record_attention=False,
                          first_token=first_token)
            tok = res.first_token
            torch.cuda.synchronize()
            ttft = time.perf_counter() - t0
            report.requests.append(_metrics(rec, k, 0, total, total, 0, 0, total * L, 0.0, ttft, 1.0, tok))
            continue
        if policy == "exact_prefix":
            keys = _prefix_keys(chunk_tokens)
            hits = 0
            while hits < k and registry.get(keys[hits]) is not None:
                hits += 1
            segs = [Segment(tokens=t, cache=registry.get(keys[i])) if i < hits else Segment(tokens=t)
                    for i, t in enumerate(chunk_tokens)]
            req = build_request(segs, question)
            res = prefill(model, req, stats=False, record_attention=False, first_token=first_token)
            tok = res.first_token
            torch.cuda.synchronize()
            ttft = time.perf_counter() - t0
            for i in range(hits, k):
                registry.put(keys[i], extract_chunk_cache(res, *req.segment_slots[i]))
            reused = sum(t.size for t in chunk_tokens[:hits])
            # (exact prefix reuse: the reused rows are the fresh run's own, deviation 0 up to rounding)
            dev = _deviation(res.hidden[slice(*res.question_span)], oracle_q) if oracle_q is not None else 0.0
            report.requests.append(_metrics(rec, k, hits, total, total - reused, reused, 0, sum(res.active_per_layer),
                                            dev, ttft, (k - hits) / k if k else 1.0, tok))
            continue
        if tier_cfg is not None and tier_pool is not None:
            # real tiers: the reference's f_r-banded placement, applied by
            # moving payloads between HBM / pinned host / disk, then the
            # disk reads of this request's hits start while it plans
            tier_pool.apply_placement(store, _tier_names(place_and_migrate(store.variants(), tier_cfg), tier_cfg))
        if policy == "cachecraft":
            plan = build_plan(chunk_tokens, question, store, alpha, focus_window, cfo_override=cfo_override)
        else:
            plan = _naive_plan(chunk_tokens, hashes, question, store, alpha)
        if tier_pool is not None:
            tier_pool.prefetch(plan)
        res, plan, req = _execute_planned(model, plan, hashes, store,
                                          use_focus=(policy == "cachecraft" and use_focus), first_token=first_token,
                                          two_pass=two_pass)
        tok = res.first_token
        torch.cuda.synchronize()
        ttft = time.perf_counter() - t0
        cfos = [cp.cfo if cp.status == HIT else 1.0 for cp in plan.chunks]
        dev = _deviation(res.hidden[slice(*res.question_span)], oracle_q) if oracle_q is not None else 0.0
        computed = plan.tokens_recomputed()
        report.requests.append(_metrics(
            rec, k, plan.hit_count, total, computed, sum(cp.n_tokens for cp in plan.chunks if cp.status == HIT),
            sum(int(cp.recompute.size) for cp in plan.chunks if cp.status == HIT and cp.recompute is not None),
            sum(res.active_per_layer), dev, ttft, float(np.mean(cfos)) if cfos else 1.0, tok))
    return report


def _metrics(rec, k, hits, total, computed, hit_total, hit_recomputed, token_layers, dev, ttft, mean_cfo, tok):
    return RequestMetrics(request_id=rec.request_id, arrival_s=rec.arrival_s, k=k, hits=hits, tokens_total=total,
                          tokens_computed=computed, tokens_reused=total - computed,
                          recompute_fraction=computed / total if total else 0.0, tokens_hit_total=hit_total,
                          tokens_hit_recomputed=hit_recomputed, token_layers=token_layers, deviation=dev, ttft=ttft,
                          mean_cfo=mean_cfo, first_token=tok)


def _tier_names(placement: dict, tier_cfg) -> dict:
    """Map the caller's tier names (ordered fastest first) onto the real
    tiers: the first is HBM, the second pinned host memory, any slower one
    disk."""
    from .tiers import DISK, HBM, HOST

    real = {t.name: (HBM, HOST)[i] if i < 2 else DISK for i, t in enumerate(tier_cfg.tiers)}
    return {vid: real[name] for vid, name in placement.items()}


def replay(trace: Trace, model_cfg=None, store_cfg=None, tier_cfg=None, alpha: float = 1.0,
           policy: str = "cachecraft", warmup: int = DEFAULT_WARMUP, queue_wait: float = DEFAULT_QUEUE_WAIT,
           focus_window: int = 3, use_focus: bool = True) -> Report:
    """The reference's replay entry point (harness.py:464-591) on the GPU:
    builds the model (``model_cfg``, default the reference's toy config, fp64
    mode) and an empty store (``store_cfg``), then replays every request of
    the trace under ``policy`` with measured TTFT.  With ``tier_cfg`` the
    variants are placed by ``place_and_migrate`` on the real tiers before
    each request (first tier HBM, second pinned host, slower ones disk) and
    disk hits are prefetched.  ``queue_wait`` is accepted for signature
    compatibility: the requests here are not queued (measured, not
    simulated, TTFT)."""
    from .model import ModelConfig, build_model
    from .store import StoreConfig, VariantStore
    from .tiers import TieredPool

    if policy not in POLICIES:
        raise ArgumentError(f"unknown policy {policy!r}; expected one of {POLICIES}")
    if queue_wait < 0:
        raise ArgumentError("queue wait must be non-negative")
    model = build_model(model_cfg or ModelConfig())
    store = VariantStore(store_cfg or StoreConfig())
    pool = None
    if tier_cfg is not None:
        tier_cfg.validate()
        pool = TieredPool(model)
    return replay_gpu(trace, model, store, alpha=alpha, policy=policy, warmup=warmup, focus_window=focus_window,
                      use_focus=use_focus, tier_cfg=tier_cfg, tier_pool=pool)
