"""Tiered chunk-cache pool on the device: a fix-up
prefill whose HIT caches live in pinned host memory (layer-wise copy-engine
preload into an L_p + 1 slot HBM ring) or on disk (async read into the host
tier) returns exactly the bits of the all-HBM run; migration round trips are
lossless; store placement follows place_and_migrate."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2502_15734_b200 as cc

    cc._native.lib()
    return cc


def _setup(cc, dtype, kw, lengths, seed):
    model = cc.build_model(cc.ModelConfig(dtype=dtype, **kw))
    r = np.random.default_rng(seed)
    vocab = kw.get("vocab_size", 256)
    chunks = [r.integers(0, vocab, n) for n in lengths]
    q = r.integers(0, vocab, 12)
    req0 = cc.plain_request(*chunks, [])
    res0 = cc.prefill(model, req0)
    caches = [cc.extract_chunk_cache(res0, s, e) for s, e in req0.segment_slots]
    caches = [cc.pad_to_blocks(c)[0] for c in caches]
    masks = [r.uniform(size=c.size) < 0.2 for c in chunks]
    return model, chunks, q, caches, masks


def _run(cc, model, chunks, q, caches, masks, **opts):
    segs = [cc.Segment(tokens=c, cache=k, recompute=m) for c, k, m in zip(chunks, caches, masks)]
    res = cc.prefill(model, cc.build_request(segs, q), first_token=True, **opts)
    torch.cuda.synchronize()
    return res


LLAMA = dict(n_layers=3, n_heads=8, d_model=512, d_head=64, vocab_size=512, rpe_base=500000.0, seed=4,
             n_kv_heads=2, d_ff=1024, mlp="swiglu", norm_weight=True, rms_eps=1e-5)


@pytest.mark.parametrize("dtype,kw,lengths", [("fp64", {}, (32, 26, 40)), ("bf16", LLAMA, (64, 48, 80)),
                                              ("fp32", LLAMA, (64, 48, 80))])
@pytest.mark.parametrize("rate", [1e15, 1e6])  # preload depth 1 (2-slot ring, recycled) / depth L
def test_host_tier_prefill_bit_identical(cc, dtype, kw, lengths, rate):
    from paper_2502_15734_b200 import tiers as T

    model, chunks, q, caches, masks = _setup(cc, dtype, kw, lengths, 5)
    ref = _run(cc, model, chunks, q, caches, masks)
    tp = T.TieredPool(model)
    host = [c.copy() for c in caches]
    for c in host[::2]:  # mixed: chunks 0 and 2 on the host tier, 1 in HBM
        tp.move(c, T.HOST)
    assert [T.tier_of(c) for c in host] == [T.HOST, T.HBM, T.HOST]
    model.h2d_bytes_per_s = rate
    got = _run(cc, model, chunks, q, host, masks)
    assert np.array_equal(got.hidden, ref.hidden)
    for l in range(model.config.n_layers):
        assert np.array_equal(got.kv.keys[l], ref.kv.keys[l])
        assert np.array_equal(got.kv.values[l], ref.kv.values[l])
    assert got.first_token == ref.first_token


def test_disk_tier_prefetch_and_round_trip(cc, tmp_path):
    from paper_2502_15734_b200 import tiers as T

    model, chunks, q, caches, masks = _setup(cc, "bf16", LLAMA, (64, 48, 80), 9)
    ref = _run(cc, model, chunks, q, caches, masks)
    tp = T.TieredPool(model, disk_dir=str(tmp_path))
    moved = [c.copy() for c in caches]
    for c in moved:
        tp.move(c, T.DISK)
    assert all(T.tier_of(c) == T.DISK for c in moved)
    for c in moved:
        c._payload.prefetch()  # asynchronous preloading while "queued"
    got = _run(cc, model, chunks, q, moved, masks)
    assert np.array_equal(got.hidden, ref.hidden)
    # disk -> host -> HBM round trip is lossless
    back = caches[1].copy()
    tp.move(back, T.DISK)
    tp.move(back, T.HBM)
    assert T.tier_of(back) == T.HBM
    for l in range(model.config.n_layers):
        assert np.array_equal(back.keys[l], caches[1].keys[l])


def test_store_placement_migrates_variants(cc):
    from paper_2502_15734_b200 import tiers as T

    model, chunks, q, caches, masks = _setup(cc, "bf16", LLAMA, (64, 48, 80), 3)
    store = cc.VariantStore(cc.StoreConfig(max_chunks=8, variants_per_chunk=2))
    ids = []
    for i, c in enumerate(caches):
        ids.append(store.insert(f"c{i}", prefix=cc.PrefixContext((), ()), a_bar=0.1, b_bar=0.1, cci=0.5,
                                token_scores=np.zeros(c.n_tokens), cache=c))
    store.touch(ids[2], 0.1)  # most reused -> fast tier
    cfg = T.TierConfig(tiers=(T.Tier("hbm", 3e12, placement_fraction=0.34), T.Tier("host", 5e10)), n_layers=3,
                       t_prefill_layer=1e-3)
    placement = T.place_and_migrate(list(store._by_id.values()), cfg)
    assert placement[ids[2]] == "hbm"
    T.TieredPool(model).apply_placement(store, placement)
    for vid, tier in placement.items():
        assert T.tier_of(store.get(vid).cache) == tier


def test_demote_slow_hits_uses_the_measured_load_rate(cc):
    """A host-tier HIT is demoted to a fresh MISS only when streaming its K/V
    over the host link would take longer than recomputing the chunk; HBM hits
    are never demoted (reference fallback_decision, tiers.py:260-299, on the
    real tiers)."""
    from paper_2502_15734_b200 import tiers
    from paper_2502_15734_b200.planner import HIT, MISS

    model, chunks, q, caches, masks = _setup(cc, "bf16", LLAMA, (64, 48, 80), 5)
    store = cc.VariantStore(cc.StoreConfig())
    for c, k in zip(chunks, caches):
        store.insert(cc.chunk_hash(c), prefix=cc.PrefixContext((), ()), a_bar=0.0, b_bar=1.0, cci=0.5,
                     token_scores=np.zeros(c.size), cache=k)
    plan = cc.build_plan(chunks, q, store, alpha=1.0)
    assert [cp.status for cp in plan.chunks] == [HIT] * 3
    pool = tiers.TieredPool(model)
    pool.to_host(plan.chunks[1].cache)
    model.h2d_bytes_per_s = 1e13  # a link fast enough that loading beats recomputing
    kept = tiers.demote_slow_hits(plan, model)
    assert [cp.status for cp in kept.chunks] == [HIT] * 3
    model.h2d_bytes_per_s = 1e3  # a pathological link: recompute instead
    out = tiers.demote_slow_hits(plan, model)
    assert [cp.status for cp in out.chunks] == [HIT, MISS, HIT]
    assert out.chunks[1].cache is None and out.chunks[1].n_slots == chunks[1].size
    res = cc.prefill(model, cc.plan_to_request(out), first_token=True)
    assert res.active_per_layer[0] == chunks[1].size + q.size + sum(
        cp.recompute.size for cp in out.chunks if cp.status == HIT and cp.recompute is not None)
