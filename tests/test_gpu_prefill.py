"""End-to-end parity of the device fix-up prefill against the reference's
golden fixtures and the CPU oracle.

Tolerances (north star): fp64 mode ~1e-9 absolute (the reference's own
precision); fp32 mode 1e-3 relative; bf16 mode relative Frobenius error
below BF16_TOY_TOL (3x the measured error) plus an identical greedy next
token.
Selections and plan decisions are bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from ccb_helpers import golden_path, record_measurement  # noqa: E402

from oracle import cachecraft_oracle as O  # noqa: E402


# bf16 mode against the float64 reference WITH UNROUNDED weights (the error
# includes rounding the weights to bf16): ~3x the largest relative error
# measured on the B200 over these small-model tests
# (profiles/r2_parity_small.jsonl: hidden / K / V 3.1e-3 - 5.1e-3); the
# full-size tests in test_gpu_parity_fullsize.py compare against the
# bf16-rounded weights
BF16_TOY_TOL = 1.5e-2
# creation statistics in bf16 (measured: token scores 1.0e-4, a/b means
# 3.6e-5 relative)
BF16_SCORE_TOL = 5e-4


@pytest.fixture(scope="module")
def cc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2502_15734_b200 as cc

    cc._native.lib()
    return cc


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# ---------------------------------------------------------------------------
# toy model, reference fixture (tests/test_model.py idioms)
# ---------------------------------------------------------------------------


def toy_result(cc, dtype="fp64"):
    g = np.load(golden_path("toy_prefill.npz"))
    model = cc.build_model(cc.ModelConfig(dtype=dtype))
    chunks = [g["c0"], g["c1"], g["c2"]]
    req0 = cc.plain_request(*chunks, [])
    res0 = cc.prefill(model, req0)
    caches = [cc.extract_chunk_cache(res0, s, e) for s, e in req0.segment_slots]
    padded, pad = cc.pad_to_blocks(caches[2])
    assert pad == 6
    segs = [
        cc.Segment(tokens=chunks[0], cache=caches[0], recompute=np.eye(32, dtype=bool)[7]),
        cc.Segment(tokens=chunks[1], cache=caches[1], recompute=g["mask1"], recompute_depth=g["depth1"]),
        cc.Segment(tokens=chunks[2], cache=padded),
    ]
    req = cc.build_request(segs, g["question"])
    return g, model, req, cc.prefill(model, req, record_attention=True, first_token=True)


def test_toy_fix_up_matches_reference_fp64(cc):
    g, model, req, res = toy_result(cc)
    assert res.active_per_layer == g["active_per_layer"].tolist()
    np.testing.assert_array_equal(res.computed, g["computed"])
    np.testing.assert_array_equal(res.positions, g["positions"])
    np.testing.assert_allclose(res.hidden, g["hidden"], atol=1e-9, rtol=0)
    for l in range(4):
        np.testing.assert_allclose(res.kv.keys[l], g[f"k{l}"], atol=1e-9, rtol=0)
        np.testing.assert_allclose(res.kv.values[l], g[f"v{l}"], atol=1e-9, rtol=0)
        np.testing.assert_allclose(res.attn.weights[l], g[f"attn{l}"], atol=1e-12, rtol=0)
        np.testing.assert_array_equal(res.attn.query_slots[l], g[f"rows{l}"])
    assert res.first_token == int(g["first_token"])
    np.testing.assert_allclose(model.logits(res.hidden[req.question_span[1] - 1])[0], g["logits_last"], atol=1e-9)


def test_bf16_mode_rejects_shapes_without_tensor_core_kernels(cc):
    """The reference's toy model (d 64, d_head 16) has no tcgen05 tiling:
    bf16 mode refuses it up front instead of silently running a slower
    kernel; the parity modes run it."""
    with pytest.raises(cc.ConfigError, match="tcgen05"):
        cc.build_model(cc.ModelConfig(dtype="bf16"))
    assert cc.ModelConfig(dtype="fp32").tensor_core_shape_error() == "d_head 16 not in (64, 128)"
    assert cc.ModelConfig.llama3_8b(n_layers=1).tensor_core_shape_error() is None
    assert cc.ModelConfig.llama3_70b(n_layers=1).tensor_core_shape_error() is None


@pytest.mark.parametrize("dtype,tol", [("fp32", 1e-3)])
def test_toy_fix_up_low_precision(cc, dtype, tol):
    g, model, req, res = toy_result(cc, dtype)
    e = {"hidden": rel(res.hidden, g["hidden"]),
         "keys": max(rel(res.kv.keys[l], g[f"k{l}"]) for l in range(4)),
         "values": max(rel(res.kv.values[l], g[f"v{l}"]) for l in range(4))}
    record_measurement("toy_fix_up", {"dtype": dtype, **e})
    for k, v in e.items():
        assert v < tol, (k, e)
    assert res.first_token == int(g["first_token"])


def test_reference_invariants_fp64(cc):
    """tests/test_model.py:145-198 + :242-255 on the device engine."""
    model = cc.build_model(cc.ModelConfig())
    r = np.random.default_rng(1234)
    chunk = r.integers(0, 256, 16)
    q = r.integers(0, 256, 4)
    req0 = cc.plain_request(r.integers(0, 256, 24), chunk, [])
    res0 = cc.prefill(model, req0)
    cache = cc.extract_chunk_cache(res0, *req0.segment_slots[1])
    stale = cache.copy()
    mask = np.zeros(16, bool)
    mask[[2, 5, 11]] = True
    res = cc.prefill(model, cc.build_request([cc.Segment(tokens=chunk, cache=cache, recompute=mask)], q))
    for layer in range(1, 4):
        changed = np.any(res.kv.keys[layer][:16] != stale.keys[layer], axis=1)
        assert np.array_equal(changed, mask)
    # layer-0 K of a recomputed row depends only on its embedding: bit-identical (M-invariant GEMM)
    assert not np.any(res.kv.keys[0][:16] != stale.keys[0])
    depth = np.full(16, 2)
    res = cc.prefill(model, cc.build_request(
        [cc.Segment(tokens=chunk, cache=cache, recompute=np.ones(16, bool), recompute_depth=depth)], q))
    assert res.active_per_layer == [20, 20, 4, 4]
    assert np.array_equal(res.kv.keys[2][:16], stale.keys[2])
    assert not np.array_equal(res.kv.keys[1][:16], stale.keys[1])


def test_garbage_caches_full_recompute_and_errors(cc):
    model = cc.build_model(cc.ModelConfig())
    r = np.random.default_rng(3)
    chunks = [r.integers(0, 256, 16) for _ in range(2)]
    q = r.integers(0, 256, 8)
    garbage = [cc.ChunkCache(keys=[r.standard_normal((16, 64)) for _ in range(4)],
                             values=[r.standard_normal((16, 64)) for _ in range(4)], n_tokens=16) for _ in chunks]
    oracle = cc.prefill(model, cc.plain_request(*chunks, q))
    reuse = cc.prefill(model, cc.build_request(
        [cc.Segment(tokens=c, cache=gc, recompute=np.ones(16, bool)) for c, gc in zip(chunks, garbage)], q))
    assert np.max(np.abs(reuse.hidden - oracle.hidden)) < 1e-9
    bad = cc.ChunkCache(keys=[np.zeros((4, 64))] * 2, values=[np.zeros((4, 64))] * 2, n_tokens=4)
    with pytest.raises(cc.PlanError):
        cc.prefill(model, cc.build_request([cc.Segment(tokens=r.integers(0, 256, 4), cache=bad)], [1]))
    with pytest.raises(cc.PlanError):
        cc.build_request([], [])


def test_pads_consume_no_positions_and_get_zero_attention(cc):
    model = cc.build_model(cc.ModelConfig())
    r = np.random.default_rng(11)
    chunk = r.integers(0, 256, 10)
    req0 = cc.plain_request(chunk, [])
    cache = cc.extract_chunk_cache(cc.prefill(model, req0), 0, 10)
    padded, pad = cc.pad_to_blocks(cache)
    assert pad == 6
    res = cc.prefill(model, cc.build_request([cc.Segment(tokens=chunk, cache=padded)], r.integers(0, 256, 5)),
                     record_attention=True)
    assert list(res.positions[:10]) == list(range(10))
    assert list(res.positions[16:]) == list(range(10, 15))
    for layer in range(4):
        assert np.all(res.attn.weights[layer][:, :, 10:16] == 0.0)
        np.testing.assert_allclose(res.attn.weights[layer].sum(axis=2), 1.0, atol=1e-12)


def test_decode_after_reuse_matches_plain(cc):
    model = cc.build_model(cc.ModelConfig())
    r = np.random.default_rng(1234)
    chunks = [r.integers(0, 256, 32) for _ in range(3)]
    q = r.integers(0, 256, 12)
    req0 = cc.plain_request(*chunks, [])
    res0 = cc.prefill(model, req0)
    caches = [cc.extract_chunk_cache(res0, s, e) for s, e in req0.segment_slots]
    oracle = cc.prefill(model, cc.plain_request(*chunks, q))
    reuse = cc.prefill(model, cc.build_request([cc.Segment(tokens=c, cache=k) for c, k in zip(chunks, caches)], q))
    o, rr = oracle.hidden[slice(*oracle.question_span)], reuse.hidden[slice(*reuse.question_span)]
    assert np.linalg.norm(rr - o) / np.linalg.norm(o) < 1e-4
    a = cc.decode(model, oracle.kv.copy(), oracle.hidden[oracle.question_span[1] - 1], 4)
    b = cc.decode(model, reuse.kv.copy(), reuse.hidden[reuse.question_span[1] - 1], 4)
    assert a == b and len(a) == 4


# ---------------------------------------------------------------------------
# BASELINE config 1 (L=2, d=256, H=4, 5 x 128 + 32, 15% recompute)
# ---------------------------------------------------------------------------


def config1_device(cc, dtype):
    g = np.load(golden_path("config1.npz"))
    model = cc.build_model(cc.ModelConfig(n_layers=2, n_heads=4, d_model=256, dtype=dtype))
    caches, scores, meta = [], [], []
    for c, oth in zip(g["chunks"], g["others"]):
        req = cc.plain_request(oth[0], oth[1], c, [])
        res = cc.prefill(model, req, stats=True)
        st = cc.creation_stats(res, ["a", "b", "c"], [2])
        prefix, a_bar, b_bar, sc = st[2]
        caches.append(cc.extract_chunk_cache(res, *req.segment_slots[2]))
        scores.append(sc.cpu().numpy())
        meta.append([a_bar, b_bar, cc.cci(a_bar, b_bar), *prefix.weights])
    return g, model, caches, scores, meta


@pytest.mark.parametrize("dtype", ["fp64", "fp32", "bf16"])
def test_config1_creation_stats_and_selection(cc, dtype):
    g, model, caches, scores, meta = config1_device(cc, dtype)
    tol = {"fp64": 1e-10, "fp32": 1e-3, "bf16": BF16_SCORE_TOL}[dtype]
    e = {"scores": rel(np.stack(scores), g["scores"]), "meta": rel(np.array(meta)[:, :2], g["meta"][:, :2])}
    sel = [cc.select_tokens(s, 0.15) for s in scores]
    flips = sum(len(set(a.tolist()) ^ set(b.tolist())) // 2 for a, b in zip(sel, g["selected"]))
    record_measurement("config1_creation", {"dtype": dtype, **e, "flips": flips,
                                            "selected": int(sum(len(s) for s in g["selected"]))})
    assert e["scores"] < tol and e["meta"] < tol, e
    if dtype != "bf16":
        np.testing.assert_array_equal(np.stack(sel), g["selected"])
    else:
        # bf16 scores may flip a selection only at a near-tie of the oracle's scores
        for s_o, got, want in zip(g["scores"], sel, g["selected"]):
            diff = set(got.tolist()) ^ set(want.tolist())
            if diff:
                kth = np.sort(s_o)[::-1][len(want) - 1]
                assert all(abs(s_o[i] - kth) < 3 * e["scores"] * abs(kth) for i in diff)


@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-9), ("fp32", 1e-3), ("bf16", BF16_TOY_TOL)])
def test_config1_fix_up_matches_reference(cc, dtype, tol):
    g, model, caches, _, _ = config1_device(cc, dtype)
    segs = []
    for c, k, idx in zip(g["chunks"], caches, g["selected"]):
        m = np.zeros(128, bool)
        m[idx] = True
        segs.append(cc.Segment(tokens=c, cache=k, recompute=m))
    req = cc.build_request(segs, g["question"])
    res = cc.prefill(model, req, first_token=True)
    q0, q1 = req.question_span
    rows = g["kv_rows"]
    e = {"hidden_q": rel(res.hidden[q0:q1], g["hidden_q"]),
         "keys": max(rel(res.kv.keys[l][rows], g[f"k{l}"]) for l in range(2)),
         "values": max(rel(res.kv.values[l][rows], g[f"v{l}"]) for l in range(2))}
    record_measurement("config1_fix_up", {"dtype": dtype, **e})
    if dtype == "fp64":
        np.testing.assert_allclose(res.hidden[q0:q1], g["hidden_q"], atol=tol)
    else:
        assert e["hidden_q"] < tol, e
    assert e["keys"] < max(tol, 1e-12) and e["values"] < max(tol, 1e-12), e
    assert res.first_token == int(g["first_token"])
    assert res.active_per_layer == g["active_per_layer"].tolist()


# ---------------------------------------------------------------------------
# Llama-shaped small model (GQA, SwiGLU, norm weights, theta 5e5) vs oracle
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-9), ("fp32", 1e-3), ("bf16", BF16_TOY_TOL)])
def test_llama_shaped_fix_up_vs_oracle(cc, dtype, tol):
    kw = dict(n_layers=3, n_heads=8, d_model=512, d_head=64, vocab_size=512, rpe_base=500000.0, seed=4,
              n_kv_heads=2, d_ff=1024, mlp="swiglu", norm_weight=True, rms_eps=1e-5)
    model = cc.build_model(cc.ModelConfig(dtype=dtype, **kw))
    ocfg = O.OracleConfig(**kw)
    w = O.draw_weights(ocfg)
    r = np.random.default_rng(8)
    chunks = [r.integers(0, 512, n) for n in (64, 48, 80)]
    q = r.integers(0, 512, 16)
    # creation on device and on the oracle (each from its own fresh prefill)
    req0 = cc.plain_request(*chunks, [])
    res0 = cc.prefill(model, req0)
    caches = [cc.extract_chunk_cache(res0, s, e) for s, e in req0.segment_slots]
    lay0 = O.layout([{"tokens": c} for c in chunks], [])
    o0 = O.prefill(w, ocfg, lay0, [None] * 3)
    ocaches = [([k[s:e] for k in o0["keys"]], [v[s:e] for v in o0["values"]]) for s, e in lay0["segment_slots"]]
    masks = [r.uniform(size=c.size) < 0.2 for c in chunks]
    segs = [cc.Segment(tokens=c, cache=k, recompute=m) for c, k, m in zip(chunks, caches, masks)]
    res = cc.prefill(model, cc.build_request(segs, q), first_token=True)
    lay = O.layout([{"tokens": c, "n_slots": c.size, "recompute": m} for c, m in zip(chunks, masks)], q)
    ref = O.prefill(w, ocfg, lay, ocaches)
    e = {"hidden": rel(res.hidden, ref["hidden"]),
         "keys": max(rel(res.kv.keys[l], ref["keys"][l]) for l in range(3)),
         "values": max(rel(res.kv.values[l], ref["values"][l]) for l in range(3))}
    record_measurement("llama_small_fix_up", {"dtype": dtype, **e})
    if dtype == "fp64":
        np.testing.assert_allclose(res.hidden, ref["hidden"], atol=tol)
    else:
        assert e["hidden"] < tol, e
    assert e["keys"] < max(tol, 1e-12) and e["values"] < max(tol, 1e-12), e
    assert res.first_token == O.greedy_token(w, ocfg, ref)


def test_programmatic_dependent_launch_is_bit_identical(cc):
    """The prefill chain launched with programmatic dependent launch
    (griddepcontrol: prologues and first weight tiles before the wait) gives
    the same bits as plain stream-ordered launches; the first token comes
    back through the pinned-copy + event path either way."""
    kw = dict(n_layers=3, n_heads=8, d_model=512, d_head=64, vocab_size=512, rpe_base=500000.0, seed=4,
              n_kv_heads=2, d_ff=1024, mlp="swiglu", norm_weight=True, rms_eps=1e-5)
    model = cc.build_model(cc.ModelConfig(dtype="bf16", **kw))
    r = np.random.default_rng(12)
    chunks = [r.integers(0, 512, n) for n in (160, 96, 200)]
    q = r.integers(0, 512, 12)
    req0 = cc.plain_request(*chunks, [])
    res0 = cc.prefill(model, req0)
    caches = [cc.extract_chunk_cache(res0, s, e) for s, e in req0.segment_slots]
    masks = [r.uniform(size=c.size) < 0.2 for c in chunks]
    segs = [cc.Segment(tokens=c, cache=k, recompute=m) for c, k, m in zip(chunks, caches, masks)]
    outs = []
    for pdl in (False, True):
        model.prefill_pdl = pdl
        res = cc.prefill(model, cc.build_request(segs, q), first_token=True)
        outs.append((res.hidden.copy(), [k.copy() for k in res.kv.keys], res.first_token))
    assert np.array_equal(outs[0][0], outs[1][0])
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)
    assert outs[0][2] == outs[1][2]
