"""Parity against the float64 CPU oracle AT THE BENCHMARKED SHAPES
(BASELINE configs 2, 4 and 5; reference model.py:348-442, :94-95,
planner.py:17-34, harness.py:331-354).

Config 2 (Llama-3-8B width: d 4096, 32/8 heads, d_ff 14336, vocab 128256,
theta 5e5; 2 of the 32 layers to bound the oracle's time):

* creation: each of the 10 x 512-token chunks is prefilled fresh behind a
  256-token prefix on the GPU (K8 creation statistics) and in the oracle;
  the token scores agree and K9 picks the 15% (77 tokens per chunk) from the
  GPU scores; the selection is compared with the oracle's selection from
  the oracle's scores (fp32: identical; bf16: flip rate measured and
  bounded);
* fix-up: the config-2 request (10 x 512 + 32 question, the oracle's
  selection, the GPU-created caches) through ``prefill(first_token=True)``
  vs ``oracle.prefill`` on the same caches: hidden, K, V of every layer and
  the last row's logits (full 128256 vocab) within 1e-3 relative in fp32
  mode and within the stated bf16 tolerance in bf16 mode; identical greedy
  token in both modes.

Config 4 (one Llama-3-70B tensor-parallel rank slice of 8: 8 q heads, 1 kv
head, 3584 MLP columns, d 8192; 1 layer; 16 x 1024 + 32 slots, 154 rows
recomputed per chunk) and config 5 (Llama-3-8B width, 1 layer, 64 x 512 + 32
= 32800 slots, 77 rows per chunk): K/V of every row and the hidden state of
a sample of the recomputed rows (the oracle evaluates the last layer's
attention only for the sampled rows; each row's output depends on its own
attention row only).

bf16 tolerances are about 3x the errors measured on the B200
(profiles/r2_parity_fullsize.jsonl, written by these tests when
CCB_PARITY_OUT is set).
"""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from ccb_helpers import (  # noqa: E402
    oracle_config,
    oracle_logits,
    oracle_weights,
    record_measurement,
    rel_err,
    row_rel_err,
)
from oracle import cachecraft_oracle as O  # noqa: E402

RATIO = 0.15
FP32_TOL = 1e-3  # north_star: 1e-3 relative in fp32 mode
# bf16 mode: ~3x the measured relative error of each quantity on the B200
# (measured, profiles/r2_parity_fullsize.jsonl: hidden 2.2e-3, K/V 1.1e-3,
# logits 2.1e-3, worst row 3.7e-3 at config 2; 1.5e-3 / 0.9e-3 at configs 4, 5)
BF16_TOL = {"hidden": 7e-3, "keys": 3.5e-3, "values": 3.5e-3, "logits": 6.5e-3, "row": 1.2e-2}
# selection flips / selected tokens with creation scores from bf16 prefills
# (measured: 0 of 770, score error 6e-5 relative)
BF16_MAX_FLIP_RATE = 0.01


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


# ---------------------------------------------------------------------------
# config 2
# ---------------------------------------------------------------------------


@functools.lru_cache(maxsize=None)
def _config2(dtype):
    import paper_2502_15734_b200 as cc

    cfg = cc.ModelConfig.llama3_8b(n_layers=2, dtype=dtype, seed=0)
    model = cc.build_model(cfg)
    r = np.random.default_rng(2502)
    V = cfg.vocab_size
    chunks = [r.integers(0, V, 512) for _ in range(10)]
    prefixes = [r.integers(0, V, 256) for _ in range(10)]
    question = r.integers(0, V, 32)
    w, remap = oracle_weights(model, chunks + prefixes + [question])
    ocfg = oracle_config(model)

    # creation (MISS path): GPU prefill with K8 stats, oracle prefill with weights
    gpu_scores, ora_scores, caches = [], [], []
    for p, c in zip(prefixes, chunks):
        req = cc.plain_request(p, c, [])
        res = cc.prefill(model, req, stats=True, record_attention=False)
        st = cc.creation_stats(res, ["p", "c"], [1])
        gpu_scores.append(st[1][3])
        caches.append(cc.extract_chunk_cache(res, *req.segment_slots[1]))
        lay = O.layout([{"tokens": remap(p)}, {"tokens": remap(c)}], [])
        ores = O.prefill(w, ocfg, lay, [None, None])
        ora_scores.append(O.fresh_chunk_stats(ores, lay["segment_slots"], ["p", "c"], 1)[4])
        del ores
    counts = [O.recompute_count(512, RATIO)] * 10
    gpu_sel = cc.planner.select_tokens_batched(gpu_scores, counts)  # K9, one launch
    ora_sel = [O.select_tokens(s, RATIO) for s in ora_scores]
    gpu_scores_h = [s.cpu().numpy() for s in gpu_scores]

    # fix-up: the oracle's selection on both sides, the GPU-created caches on both sides
    masks = []
    for sel in ora_sel:
        m = np.zeros(512, bool)
        m[sel] = True
        masks.append(m)
    segs = [cc.Segment(tokens=c, cache=k, recompute=m) for c, k, m in zip(chunks, caches, masks)]
    req = cc.build_request(segs, question)
    res = cc.prefill(model, req, record_attention=False, stats=False, first_token=True)
    ocaches = [(k.keys, k.values) for k in caches]
    lay = O.layout([{"tokens": remap(c), "n_slots": k.n_slots, "recompute": m}
                    for c, k, m in zip(chunks, caches, masks)], remap(question))
    ref = O.prefill(w, ocfg, lay, ocaches, keep_weights=False)
    q1 = req.question_span[1]
    ref_logits = oracle_logits(model, ref["hidden"][q1 - 1])
    out = {
        "model": model, "req": req, "ref": ref, "ref_logits": ref_logits,
        "hidden": res.hidden, "keys": [res.kv.keys[l] for l in range(2)],
        "values": [res.kv.values[l] for l in range(2)],
        "logits": res.extras["logits_last"].double().cpu().numpy()[0], "token": res.first_token,
        "active": res.active_per_layer, "gpu_scores": gpu_scores_h, "ora_scores": ora_scores,
        "gpu_sel": gpu_sel, "ora_sel": ora_sel, "caches": caches,
    }
    return out


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_config2_creation_scores_and_selection(dtype):
    _need_gpu()
    o = _config2(dtype)
    errs = [rel_err(g, r) for g, r in zip(o["gpu_scores"], o["ora_scores"])]
    flips = sum(int(np.setdiff1d(o["ora_sel"][i], o["gpu_sel"][i]).size) for i in range(10))
    selected = sum(s.size for s in o["ora_sel"])
    # every flip must sit at the selection boundary: the oracle's score of a
    # swapped token is within the measured score error of the k-th score
    boundary = []
    for i in range(10):
        s = o["ora_scores"][i]
        kth = np.sort(s)[::-1][o["ora_sel"][i].size - 1]
        for t in np.setxor1d(o["ora_sel"][i], o["gpu_sel"][i]):
            boundary.append(abs(s[t] - kth) / max(abs(kth), 1e-30))
    record_measurement("config2_selection", {"dtype": dtype, "score_rel_err_max": max(errs), "flips": flips,
                                             "selected": selected, "flip_rate": flips / selected,
                                             "max_flip_gap_rel": max(boundary) if boundary else 0.0})
    if dtype == "fp32":
        assert max(errs) < FP32_TOL, errs
        assert flips == 0 or max(boundary) < 10 * max(errs), (flips, boundary)
    else:
        assert max(errs) < 2e-4, errs  # measured 6.2e-5
        assert flips / selected <= BF16_MAX_FLIP_RATE, (flips, selected)
        assert max(boundary, default=0.0) < 20 * max(errs), boundary
    # K9 itself is bit-exact on identical inputs: GPU selection == oracle
    # selection applied to the GPU's own scores
    for g, s in zip(o["gpu_sel"], o["gpu_scores"]):
        assert np.array_equal(np.asarray(g), O.select_tokens(s, RATIO))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_config2_fixup_prefill_matches_oracle(dtype):
    _need_gpu()
    o = _config2(dtype)
    ref, req = o["ref"], o["req"]
    rows = np.flatnonzero(ref["computed"])
    assert o["active"] == ref["active_per_layer"] == [802, 802]
    e = {
        "hidden": rel_err(o["hidden"][rows], ref["hidden"][rows]),
        "hidden_row": row_rel_err(o["hidden"][rows], ref["hidden"][rows]),
        "keys": max(rel_err(o["keys"][l], ref["keys"][l]) for l in range(2)),
        "values": max(rel_err(o["values"][l], ref["values"][l]) for l in range(2)),
        "logits": rel_err(o["logits"], o["ref_logits"]),
    }
    top2 = np.sort(o["ref_logits"])[-2:]
    record_measurement("config2_fixup", {"dtype": dtype, **e, "token": o["token"],
                                         "oracle_token": int(np.argmax(o["ref_logits"])),
                                         "oracle_top2_gap": float(top2[1] - top2[0])})
    # cached rows of the returned KV are the injected cache rows, bit for bit
    for l in range(2):
        for (s, t), c in zip(req.segment_slots, o["caches"]):
            keep = ~req.recompute_mask[s:t]
            assert np.array_equal(o["keys"][l][s:t][keep], np.asarray(c.keys[l])[: t - s][keep])
    if dtype == "fp32":
        for k in ("hidden", "hidden_row", "keys", "values", "logits"):
            assert e[k] < FP32_TOL, (k, e)
    else:
        for k, tol in (("hidden", BF16_TOL["hidden"]), ("hidden_row", BF16_TOL["row"]), ("keys", BF16_TOL["keys"]),
                       ("values", BF16_TOL["values"]), ("logits", BF16_TOL["logits"])):
            assert e[k] < tol, (k, e)
    assert o["token"] == int(np.argmax(o["ref_logits"])), (o["token"], top2)


# ---------------------------------------------------------------------------
# configs 4 (70B TP rank slice) and 5 (32k prompt): one layer, sampled rows
# ---------------------------------------------------------------------------


def _random_caches(k, n_slots, kvw, dtype, rng):
    """Random injected caches (as the reference's garbage-cache tests do,
    tests/test_model.py:98-121), pre-rounded to the model's storage dtype so
    both sides see the same values."""
    import paper_2502_15734_b200 as cc

    out = []
    for _ in range(k):
        ks = torch.from_numpy(rng.standard_normal((1, n_slots, kvw)))
        vs = torch.from_numpy(rng.standard_normal((1, n_slots, kvw)))
        if dtype == "bf16":
            ks, vs = ks.bfloat16().double(), vs.bfloat16().double()
        elif dtype == "fp32":
            ks, vs = ks.float().double(), vs.float().double()
        out.append(cc.ChunkCache(keys=list(ks.numpy()), values=list(vs.numpy()), n_tokens=n_slots))
    return out


def _one_layer_case(model, n_chunks, chunk_len, name, dtype, seed, n_sample=192):
    import paper_2502_15734_b200 as cc

    cfg = model.kcfg
    r = np.random.default_rng(seed)
    chunks = [r.integers(0, cfg.vocab_size, chunk_len) for _ in range(n_chunks)]
    question = r.integers(0, cfg.vocab_size, 32)
    k = O.recompute_count(chunk_len, RATIO)
    masks = []
    for _ in range(n_chunks):
        m = np.zeros(chunk_len, bool)
        m[r.choice(chunk_len, k, replace=False)] = True
        masks.append(m)
    caches = _random_caches(n_chunks, chunk_len, cfg.kv_width(), dtype, r)
    segs = [cc.Segment(tokens=c, cache=kc, recompute=m) for c, kc, m in zip(chunks, caches, masks)]
    req = cc.build_request(segs, question)
    res = cc.prefill(model, req, record_attention=False, stats=False)
    w, remap = oracle_weights(model, chunks + [question])
    rows = np.flatnonzero(req.recompute_mask)
    sample = np.sort(np.concatenate([r.choice(rows[:-32], n_sample - 32, replace=False), rows[-32:]]))
    lay = O.layout([{"tokens": remap(c), "n_slots": chunk_len, "recompute": m} for c, m in zip(chunks, masks)],
                   remap(question))
    ref = O.prefill(w, oracle_config(model), lay, [(kc.keys, kc.values) for kc in caches], keep_weights=False,
                    sample_rows=sample)
    e = {
        "keys": rel_err(res.kv.keys[0], ref["keys"][0]),
        "values": rel_err(res.kv.values[0], ref["values"][0]),
        "hidden": rel_err(res.hidden[sample], ref["hidden"][sample]),
        "hidden_row": row_rel_err(res.hidden[sample], ref["hidden"][sample]),
    }
    record_measurement(name, {"dtype": dtype, "slots": req.n_slots, "recomputed": int(rows.size),
                              "sampled_rows": int(sample.size), **e})
    assert req.n_slots == n_chunks * chunk_len + 32
    assert res.active_per_layer == [n_chunks * k + 32]
    tol = {"keys": FP32_TOL, "values": FP32_TOL, "hidden": FP32_TOL, "hidden_row": FP32_TOL} if dtype == "fp32" else {
        "keys": BF16_TOL["keys"], "values": BF16_TOL["values"], "hidden": BF16_TOL["hidden"],
        "hidden_row": BF16_TOL["row"]}
    for key, t in tol.items():
        assert e[key] < t, (key, e)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_config5_32k_prompt_one_layer_matches_oracle(dtype):
    _need_gpu()
    import paper_2502_15734_b200 as cc

    model = cc.build_model(cc.ModelConfig.llama3_8b(n_layers=1, dtype=dtype, seed=5))
    _one_layer_case(model, 64, 512, "config5_32k", dtype, seed=32800)
    del model
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_config4_70b_tp_rank_slice_matches_oracle(dtype):
    """Rank 3 of a TP8 Llama-3-70B layer, run alone: with an identity
    all-reduce the rank's residual adds its own o_proj / down_proj partial
    (oracle.prefill's ``tp`` restatement with the same partial sums)."""
    _need_gpu()
    import paper_2502_15734_b200 as cc
    from paper_2502_15734_b200 import parallel

    cfg = cc.ModelConfig.llama3_70b(n_layers=1, dtype=dtype, seed=4)
    sl = parallel.tp_slices(cfg.n_heads, cfg.kv_heads(), cfg.ff_dim(), 3, 8)
    model = cc.build_model(cfg, tp=parallel.TPContext(sl, allreduce=lambda t: t))
    assert (model.kcfg.n_heads, model.kcfg.kv_heads(), model.kcfg.ff_dim()) == (8, 1, 3584)
    _one_layer_case(model, 16, 1024, "config4_70b_tp_rank", dtype, seed=70, n_sample=160)
    del model
    torch.cuda.empty_cache()
