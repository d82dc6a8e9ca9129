"""GPU replay of the reference's harness loop (harness.py:464-591) in fp64
mode: every per-request decision (hits, recomputed tokens, token-layers,
mean CFO) must equal the reference's, including focused-chunk early
termination; deviations agree to fp64 precision."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from ccb_helpers import load_json  # noqa: E402


@pytest.mark.parametrize("name,policy,focus,layers,two_pass", [
    ("cachecraft", "cachecraft", False, 2, False),
    ("full_cache_naive", "full_cache_naive", False, 2, False),
    ("cachecraft_focus", "cachecraft", True, 6, True),   # the reference's two-pass early termination
    ("cachecraft_focus", "cachecraft", True, 6, False),  # single-pass online early termination (f1)
])
def test_replay_decisions_match_reference(name, policy, focus, layers, two_pass):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2502_15734_b200 as cc
    from paper_2502_15734_b200 import harness

    g = load_json("replay.json")
    tr = harness.gen_synthetic(12, 1.2, 3, 14, chunk_len_range=(16, 40), seed=3, question_len_range=(4, 8))
    model = cc.build_model(cc.ModelConfig(n_layers=layers, n_heads=4, d_model=64))
    store = cc.VariantStore(cc.StoreConfig(max_chunks=5, variants_per_chunk=3))
    rep = harness.replay_gpu(tr, model, store, alpha=1.0, policy=policy, warmup=0, use_focus=focus, focus_window=2,
                            two_pass=two_pass)
    want = g[name]
    got = [(m.hits, m.tokens_computed, m.token_layers, m.tokens_hit_recomputed) for m in rep.requests]
    assert got == [(w["hits"], w["tokens_computed"], w["token_layers"], w["hit_recomputed"]) for w in want]
    np.testing.assert_allclose([m.mean_cfo for m in rep.requests], [w["mean_cfo"] for w in want], atol=1e-9)
    np.testing.assert_allclose([m.deviation for m in rep.requests], [w["deviation"] for w in want], atol=1e-7)


def test_replay_baselines_run_and_rank():
    """Policy ordering on a small Zipf trace (tests/test_trends.py:115-153):
    full >= cachecraft computed tokens, exact-prefix deviation 0."""
    import paper_2502_15734_b200 as cc
    from paper_2502_15734_b200 import harness

    tr = harness.gen_synthetic(10, 1.2, 3, 12, chunk_len_range=(32, 48), seed=1, question_len_range=(8, 8))
    model = cc.build_model(cc.ModelConfig(n_layers=2, n_heads=4, d_model=64))
    aggs = {}
    for policy in ("full_recompute", "exact_prefix", "cachecraft"):
        st = cc.VariantStore(cc.StoreConfig(max_chunks=20, variants_per_chunk=3))
        aggs[policy] = harness.replay_gpu(tr, model, st, policy=policy, warmup=2).aggregate()
    assert aggs["full_recompute"]["tokens_computed"] >= aggs["exact_prefix"]["tokens_computed"]
    assert aggs["full_recompute"]["tokens_computed"] >= aggs["cachecraft"]["tokens_computed"]
    assert aggs["exact_prefix"]["mean_deviation"] < 1e-9


def test_online_focus_cut_keeps_recorded_attention_and_values_consistent():
    """prefill(focus_window=w, record_attention=True, record_values=True):
    when the online early termination cuts unfocused chunks mid-prefill, the
    recorded softmax weights, query slots and value traces of EVERY layer
    equal those of a prefill that runs the post-cut depths from the start
    (the reference's second pass, harness.py:425-428) — layers recorded
    before the cut keep the row order they ran in."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2502_15734_b200 as cc

    model = cc.build_model(cc.ModelConfig(n_layers=6, n_heads=4, d_model=64))
    for seed in range(40):
        r = np.random.default_rng(seed)
        chunks = [r.integers(0, 256, 24) for _ in range(4)]
        q = r.integers(0, 256, 6)
        base = cc.prefill(model, cc.plain_request(*chunks, []), record_attention=False)
        caches = [cc.extract_chunk_cache(base, s, e) for s, e in cc.plain_request(*chunks, []).segment_slots]
        masks = [r.uniform(size=24) < 0.4 for _ in chunks]
        segs = [cc.Segment(tokens=c, cache=k, recompute=m) for c, k, m in zip(chunks, caches, masks)]
        one = cc.prefill(model, cc.build_request(segs, q), record_attention=True, record_values=True, focus_window=2)
        if not one.extras.get("focus_cut"):
            continue
        focus = one.extras["focus"]
        segs2 = []
        for i, (c, k, m) in enumerate(zip(chunks, caches, masks)):
            depth = None if i in focus.focused else np.full(24, focus.cutoff_layer, np.int64)
            segs2.append(cc.Segment(tokens=c, cache=k, recompute=m, recompute_depth=depth))
        two = cc.prefill(model, cc.build_request(segs2, q), record_attention=True, record_values=True)
        assert one.active_per_layer == two.active_per_layer
        for l in range(6):
            np.testing.assert_array_equal(one.attn.query_slots[l], two.attn.query_slots[l])
            np.testing.assert_allclose(one.attn.weights[l], two.attn.weights[l], atol=1e-12, rtol=0)
            np.testing.assert_allclose(one.value_trace[l][1], two.value_trace[l][1], atol=1e-12, rtol=0)
        np.testing.assert_allclose(one.hidden, two.hidden, atol=1e-12, rtol=0)
        return
    pytest.skip("no seed produced an early-termination cut")
