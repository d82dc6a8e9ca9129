"""Generate golden fixtures from the UNMODIFIED reference package.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes small .npz / .json files next to this script.  They pin the CPU
oracle (``oracle/cachecraft_oracle.py``) and, through it, the B200 engine.
Scenario idioms follow the reference's own tests (cited per block).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")

import cachecraft as cc  # noqa: E402  (the reference)
from cachecraft.harness import _fresh_chunk_stats  # noqa: E402
from cachecraft.stats import ChunkSpan  # noqa: E402


def _save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)


def _json(name, obj):
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(obj, fh, indent=1, sort_keys=True)


def gen_rope():
    # tests/test_rpe.py idioms: rotation oracle, per-head slices, round trip
    r = np.random.default_rng(11)
    x = r.standard_normal((24, 32))
    pos = np.concatenate([np.array([0, 1, 3, 17, 255, 1024, 4095, 32767]), r.integers(0, 40000, 16)])
    _save(
        "rope.npz",
        x=x,
        pos=pos,
        apply_full=cc.apply_rpe(x, pos),
        apply_h8=cc.apply_rpe(x, pos, d_head=8),
        remove_h8=cc.remove_rpe(x, pos, d_head=8),
        apply_h16_b5e5=cc.apply_rpe(x, pos, base=500000.0, d_head=16),
    )


def gen_select():
    # tests/test_planner.py:35-70 (KATs, ties, sort oracle)
    r = np.random.default_rng(5)
    cases = [
        ([3.0, 1.0, 2.0], 0.0),
        ([3.0, 1.0], 1.0),
        ([1.0, 1.0, 1.0, 1.0], 0.5),
        (list(r.permutation(10).astype(float)), 0.3),
        ([0.0] * 7 + [1.0] * 5, 0.25),
    ]
    for n in (1, 5, 16, 64, 128, 512, 1024):
        s = r.standard_normal(n)
        s[r.integers(0, n, max(1, n // 8))] = 0.5  # planted ties
        for c in (0.0, 0.05, 0.1, 0.15, 0.2, 0.333333, 0.5, 0.999, 1.0):
            cases.append((list(map(float, s)), c))
    out = [{"scores": s, "cfo": c, "selected": [int(i) for i in cc.select_tokens(s, c)]} for s, c in cases]
    _json("select.json", out)


def gen_scoring():
    # tests/test_scoring.py KATs + random cases
    r = np.random.default_rng(9)
    ids = [f"c{i}" for i in range(8)]
    cases = []
    for _ in range(40):
        m = int(r.integers(0, 6))
        old = list(r.choice(ids, size=m, replace=False))
        new = list(r.choice(ids, size=int(r.integers(0, 7)), replace=False))
        w = [float(x) for x in r.uniform(0, 2, size=m)]
        cci_v = float(r.uniform(0.5, 1.0))
        alpha = float(r.choice([0.35, 1.0, 2.0]))
        ctx = cc.PrefixContext(chunk_ids=tuple(old), weights=tuple(w))
        sc = cc.score_variant(ctx, cci_v, new, alpha)
        cases.append(
            {"old": old, "w": w, "new": new, "cci": cci_v, "alpha": alpha,
             "beta": sc.beta, "gamma": sc.gamma, "beta_prime": sc.beta_prime, "cfo": sc.cfo}
        )
    ccis = [[a, b, cc.cci(a, b)] for a, b in [(0.25, 0.25), (1.0, 0.0), (0.0063, 0.00147), (0.5, 2.0)]]
    _json("scoring.json", {"cases": cases, "cci": ccis,
                           "cfo_kat": cc.cfo(2.0, 0.8, 0.5), "adj_kat": cc.adjusted_beta(0.75, 1 / 3)})


def gen_hash():
    r = np.random.default_rng(2)
    toks = [list(map(int, r.integers(0, 128256, n))) for n in (1, 7, 16, 128, 512)]
    _json("hash.json", [{"tokens": t, "hash": cc.chunk_hash(t)} for t in toks])


def gen_weights():
    out = []
    for kw in ({}, {"n_layers": 2, "n_heads": 4, "d_model": 256}, {"n_layers": 2, "n_heads": 2, "d_model": 32, "seed": 7}):
        m = cc.build_model(cc.ModelConfig(**kw))
        out.append({"config": kw, "blake2b": hashlib.blake2b(m.weight_bytes(), digest_size=16).hexdigest(),
                    "embed00": float(m.embed[0, 0]), "w_down_last": float(m.layers[-1].w_down[-1, -1])})
    _json("weights.json", out)


def _kv_dump(prefix, res, rows):
    d = {}
    for l in range(len(res.kv.keys)):
        d[f"{prefix}k{l}"] = res.kv.keys[l][rows]
        d[f"{prefix}v{l}"] = res.kv.values[l][rows]
    return d


def gen_toy_prefill():
    # tests/test_model.py:97-198 idioms on the toy model (L=4, H=4, d=64)
    model = cc.build_model(cc.ModelConfig())
    r = np.random.default_rng(1234)
    chunks = [r.integers(0, 256, n) for n in (32, 32, 26)]
    q = r.integers(0, 256, 12)
    req0 = cc.plain_request(*chunks, [])
    res0 = cc.prefill(model, req0)
    caches = [cc.extract_chunk_cache(res0, s, e) for s, e in req0.segment_slots]
    # partial mask + depth cap on the middle chunk, pads on the last
    mask = np.zeros(32, bool)
    mask[[2, 5, 11, 30]] = True
    depth = np.zeros(32, np.int64)
    depth[mask] = 2
    padded, _ = cc.pad_to_blocks(caches[2])
    segs = [
        cc.Segment(tokens=chunks[0], cache=caches[0], recompute=np.eye(32, dtype=bool)[7]),
        cc.Segment(tokens=chunks[1], cache=caches[1], recompute=mask, recompute_depth=depth),
        cc.Segment(tokens=chunks[2], cache=padded),
    ]
    req = cc.build_request(segs, q)
    res = cc.prefill(model, req)
    out = {
        "c0": chunks[0], "c1": chunks[1], "c2": chunks[2], "question": q, "mask1": mask, "depth1": depth,
        "hidden": res.hidden, "active_per_layer": np.array(res.active_per_layer),
        "computed": res.computed, "positions": res.positions, "is_pad": req.is_pad,
        "first_token": np.array(int(np.argmax(model.logits(res.hidden[req.question_span[1] - 1])[0]))),
        "logits_last": model.logits(res.hidden[req.question_span[1] - 1])[0],
    }
    for l in range(4):
        out[f"k{l}"], out[f"v{l}"] = res.kv.keys[l], res.kv.values[l]
        out[f"attn{l}"] = res.attn.weights[l]
        out[f"rows{l}"] = res.attn.query_slots[l]
    _save("toy_prefill.npz", **out)


def gen_stats():
    # tests/test_stats.py:61-69 prompt
    model = cc.build_model(cc.ModelConfig())
    r = np.random.default_rng(7)
    lengths = [12, 9, 15]
    chunks = [r.integers(0, 256, n) for n in lengths]
    qq = r.integers(0, 256, 6)
    res = cc.prefill(model, cc.plain_request(*chunks, qq))
    spans = cc.spans_from_lengths(range(3), lengths)
    st = cc.compute_stats(res.attn, spans)
    out = {"c0": chunks[0], "c1": chunks[1], "c2": chunks[2], "q": qq,
           "stream": cc.question_inter_stream(res.attn, spans, res.question_span)}
    for i in range(3):
        out[f"intra{i}"] = st.intra_table[i]
        out[f"diag{i}"] = st.diag_table[i]
        out[f"tok{i}"] = st.token_inter[i]
        out[f"ratios{i}"] = np.array(cc.context_ratios(st, i))
        for j in range(i):
            out[f"inter{j}_{i}"] = st.inter_table[(j, i)]
    _save("stats_toy.npz", **out)


def gen_config1():
    """BASELINE config 1: L=2, d=256, H=4, vocab 256; 5 chunks x 128 + 32
    question; caches created under random 2-chunk prefixes
    (tests/test_trends.py:54-60 idiom); fix-up at 15% via select_tokens."""
    cfg = cc.ModelConfig(n_layers=2, n_heads=4, d_model=256)
    model = cc.build_model(cfg)
    r = np.random.default_rng(2025)
    chunks = [r.integers(0, 256, 128) for _ in range(5)]
    others = [[r.integers(0, 256, 128) for _ in range(2)] for _ in range(5)]
    q = r.integers(0, 256, 32)
    caches, scores, meta = [], [], []
    for c, oth in zip(chunks, others):
        req = cc.plain_request(*oth, c, [])
        res = cc.prefill(model, req)
        spans = [ChunkSpan(i, s, e - s) for i, (s, e) in enumerate(req.segment_slots)]
        prefix, a_bar, b_bar, sc = _fresh_chunk_stats(res.attn, spans, 2)
        s0, s1 = req.segment_slots[2]
        caches.append(cc.extract_chunk_cache(res, s0, s1))
        scores.append(sc)
        meta.append([a_bar, b_bar, cc.cci(a_bar, b_bar), *prefix.weights])
    sel = [cc.select_tokens(s, 0.15) for s in scores]
    segs = []
    for c, k, idx in zip(chunks, caches, sel):
        m = np.zeros(128, bool)
        m[idx] = True
        segs.append(cc.Segment(tokens=c, cache=k, recompute=m))
    req = cc.build_request(segs, q)
    res = cc.prefill(model, req)
    full = cc.prefill(model, cc.plain_request(*chunks, q))
    q0, q1 = req.question_span
    rows = np.unique(np.concatenate([np.arange(0, req.n_slots, 16), np.flatnonzero(req.recompute_mask)]))
    out = {
        "chunks": np.stack(chunks), "others": np.array([np.stack(o) for o in others]), "question": q,
        "scores": np.stack(scores), "meta": np.array(meta), "selected": np.stack(sel),
        "hidden_q": res.hidden[q0:q1], "logits_last": model.logits(res.hidden[q1 - 1])[0],
        "first_token": np.array(int(np.argmax(model.logits(res.hidden[q1 - 1])[0]))),
        "full_hidden_q": full.hidden[q0:q1],
        "full_first_token": np.array(int(np.argmax(model.logits(full.hidden[q1 - 1])[0]))),
        "kv_rows": rows, "active_per_layer": np.array(res.active_per_layer),
    }
    out.update(_kv_dump("", res, rows))
    _save("config1.npz", **out)


def gen_plan():
    # tests/test_planner.py:148-247 idioms: seeded store, min-CFO variant, ceil count
    r = np.random.default_rng(31)
    store = cc.VariantStore(cc.StoreConfig(max_chunks=3, variants_per_chunk=3))
    chunks = [r.integers(0, 256, int(n)) for n in (8, 10, 16, 24, 9)]
    ids = [cc.chunk_hash(c) for c in chunks]
    log = []
    for rep in range(12):
        ci = int(r.integers(0, 5))
        m = int(r.integers(0, 4))
        pre = list(r.choice([x for x in ids if x != ids[ci]] + ["zz", "yy"], size=m, replace=False))
        w = [float(x) for x in r.uniform(0, 1, m)]
        n = chunks[ci].size
        tok_scores = r.standard_normal(n)
        tok_scores[r.integers(0, n, 2)] = 0.25
        cache = cc.ChunkCache(keys=[np.zeros((n, 4))], values=[np.zeros((n, 4))], n_tokens=n)
        vid = store.insert(ids[ci], prefix=cc.PrefixContext(chunk_ids=tuple(pre), weights=tuple(w)),
                           a_bar=0.1, b_bar=0.1, cci=float(r.uniform(0.5, 1.0)),
                           token_scores=tok_scores, cache=cache)
        log.append({"chunk": ci, "prefix": pre, "weights": w, "cci": store.get(vid).cci,
                    "scores": [float(x) for x in tok_scores], "vid": vid})
        if rep % 3 == 2:
            store.touch(vid, float(r.uniform(0, 1)))
            log[-1]["touched_fr"] = store.get(vid).f_r
    plans = []
    for trial in range(6):
        order = [int(x) for x in r.permutation(5)[: int(r.integers(2, 6))]]
        alpha = float(r.choice([0.35, 1.0, 3.0]))
        plan = cc.build_plan([chunks[i] for i in order], r.integers(0, 256, 4), store, alpha)
        plans.append({"order": order, "alpha": alpha, "chunks": [
            {"status": cp.status, "variant_id": cp.variant_id, "cfo": cp.cfo,
             "recompute": [] if cp.recompute is None else [int(i) for i in cp.recompute]}
            for cp in plan.chunks]})
    _json("plan.json", {"chunks": [list(map(int, c)) for c in chunks], "inserts": log, "plans": plans,
                        "live": [v.variant_id for v in store.variants()],
                        "census": store.census()})


    print("golden fixtures written to", HERE)


def gen_replay():
    """harness.py:67-144 trace synthesis + harness.py:464-591 replay at a tiny
    config (no early termination): per-request decisions to reproduce."""
    from cachecraft.harness import top_share

    tr = cc.gen_synthetic(12, 1.2, 3, 14, chunk_len_range=(16, 40), seed=3, question_len_range=(4, 8))
    skew = cc.fit_zipf_skew(60, 5, 40, target_share=0.6, seed=3, iterations=10)
    out = {"trace": [{"id": r.request_id, "chunks": list(map(int, r.chunk_ids)), "q": [int(t) for t in r.question],
                      "arrival": r.arrival_s} for r in tr.records],
           "corpus": {str(k): [int(t) for t in v] for k, v in tr.corpus.items()},
           "skew": skew, "top_share": top_share(tr)}
    cfg = cc.ModelConfig(n_layers=2, n_heads=4, d_model=64)
    for name, policy, focus in (("cachecraft", "cachecraft", False), ("full_cache_naive", "full_cache_naive", False),
                                 ("cachecraft_focus", "cachecraft", True)):
        mcfg = cc.ModelConfig(n_layers=6, n_heads=4, d_model=64) if focus else cfg
        rep = cc.replay(tr, model_cfg=mcfg, store_cfg=cc.StoreConfig(max_chunks=5, variants_per_chunk=3), alpha=1.0,
                        policy=policy, warmup=0, use_focus=focus, focus_window=2)
        out[name] = [{"hits": m.hits, "tokens_computed": m.tokens_computed, "token_layers": m.token_layers,
                        "mean_cfo": m.mean_cfo, "deviation": m.deviation, "hit_recomputed": m.tokens_hit_recomputed}
                       for m in rep.requests]
    _json("replay.json", out)




def gen_decode():
    # model.py:445-484 greedy decode continuing the toy fix-up prefill of
    # gen_toy_prefill (its KV holds pad rows: kv.valid False, position 0)
    model = cc.build_model(cc.ModelConfig())
    r = np.random.default_rng(1234)
    chunks = [r.integers(0, 256, n) for n in (32, 32, 26)]
    q = r.integers(0, 256, 12)
    req0 = cc.plain_request(*chunks, [])
    res0 = cc.prefill(model, req0)
    caches = [cc.extract_chunk_cache(res0, s, e) for s, e in req0.segment_slots]
    padded, _ = cc.pad_to_blocks(caches[2])
    segs = [cc.Segment(tokens=chunks[0], cache=caches[0], recompute=np.eye(32, dtype=bool)[7]),
            cc.Segment(tokens=chunks[1], cache=caches[1]), cc.Segment(tokens=chunks[2], cache=padded)]
    req = cc.build_request(segs, q)
    res = cc.prefill(model, req)
    kv = res.kv.copy()
    n0 = kv.positions.size
    last = res.hidden[req.question_span[1] - 1]
    toks = cc.decode(model, kv, last, 6)
    out = {"c0": chunks[0], "c1": chunks[1], "c2": chunks[2], "question": q, "tokens": np.array(toks),
           "n0": np.array(n0), "positions": kv.positions, "valid": kv.valid, "last_hidden": last}
    for l in range(4):
        out[f"k{l}"], out[f"v{l}"] = kv.keys[l], kv.values[l]
    _save("decode_toy.npz", **out)


def gen_tiers():
    # tiers.py:62-71 preload_depth and :209-261 place_and_migrate
    # (tests/test_tiers.py idioms: f_r bands, byte budgets, spill)
    from cachecraft import tiers as T

    depth = []
    for L in (1, 2, 5, 32, 80):
        for tp, tl in ((1.0, 2.0), (2.0, 1.0), (1.0, 1.0), (0.3, 0.9), (0.49, 0.38), (1e-3, 5.0)):
            depth.append({"L": L, "tp": tp, "tl": tl, "depth": T.preload_depth(L, tp, tl)})
    store = cc.VariantStore(cc.StoreConfig(max_chunks=8, variants_per_chunk=3))
    r = np.random.default_rng(17)
    vids = []
    for i in range(12):
        n = int(r.integers(8, 40))
        keys = [np.zeros((n, 8)) for _ in range(2)]
        cache = cc.ChunkCache(keys=keys, values=[k.copy() for k in keys], n_tokens=n)
        vid = store.insert(f"c{i % 7}", prefix=cc.PrefixContext((f"p{i}",), (1.0,)), a_bar=0.1, b_bar=0.1,
                           cci=0.5, token_scores=np.zeros(n), cache=cache)
        vids.append(vid)
        for _ in range(int(r.integers(0, 4))):
            store.touch(vid, float(r.uniform(0.05, 1.0)))
    variants = list(store._by_id.values())
    meta = [{"variant_id": v.variant_id, "f_r": v.f_r, "created_at": v.created_at, "bytes": v.payload_bytes()}
            for v in variants]
    cases = []
    for fracs, caps in (((0.25, 0.5, None), (None, None, None)), ((0.5, None), (20000, None)),
                        ((0.2, 0.3, None), (6000, 30000, None))):
        tiers = tuple(T.Tier(name=nm, bandwidth=bw, capacity_bytes=cp, placement_fraction=fr)
                      for nm, bw, cp, fr in zip(("hbm", "host", "disk"), (3e12, 5e10, 5e9), caps, fracs))
        cfg = T.TierConfig(tiers=tiers, n_layers=4, t_prefill_layer=1e-3)
        cases.append({"fractions": list(fracs), "capacities": list(caps),
                      "placement": {str(k): v for k, v in T.place_and_migrate(variants, cfg).items()}})
    _json("tiers.json", {"depth": depth, "variants": meta, "placement": cases})


if __name__ == "__main__":
    only = os.environ.get("GEN_ONLY")
    gens = [gen_rope, gen_select, gen_scoring, gen_hash, gen_weights, gen_toy_prefill, gen_stats, gen_config1,
            gen_plan, gen_replay, gen_decode, gen_tiers]
    for g in gens:
        if not only or g.__name__ == "gen_" + only:
            g()
