"""Variant store metadata behaviour (host logic, store.py:94-263 semantics;
idioms of the reference's tests/test_store.py).  Host-array caches only: no
GPU needed."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2502_15734_b200 import ArgumentError, ChunkCache, NotFoundError, PrefixContext, StoreConfig, VariantStore
from paper_2502_15734_b200 import chunk_hash, pad_to_blocks


def cache(n, width=8, layers=2, fill=1.0):
    return ChunkCache(keys=[np.full((n, width), fill) for _ in range(layers)],
                      values=[np.full((n, width), -fill) for _ in range(layers)], n_tokens=n)


def insert(store, cid, prefix=(), n=10):
    return store.insert(cid, prefix=PrefixContext(chunk_ids=tuple(prefix), weights=tuple(1.0 for _ in prefix)),
                        a_bar=0.1, b_bar=0.2, cci=0.6, token_scores=np.arange(n, dtype=float), cache=cache(n))


def test_chunk_hash_digest_and_raw_ids():
    assert len(chunk_hash([1, 2, 3])) == 16
    assert chunk_hash([1, 2, 3]) == chunk_hash(np.array([1, 2, 3], dtype=np.int64))
    assert chunk_hash([1, 2, 3]) != chunk_hash([1, 2, 4])
    with pytest.raises(ArgumentError):
        chunk_hash([])


def test_pad_to_blocks_seventeen_rows():
    padded, pad = pad_to_blocks(cache(17))
    assert pad == 15 and padded.n_slots == 32 and padded.n_tokens == 17
    assert np.all(padded.keys[0][17:] == 0.0)
    same, pad0 = pad_to_blocks(cache(16))
    assert pad0 == 0 and same.n_slots == 16


def test_insert_lookup_replace_and_accumulate():
    store = VariantStore(StoreConfig())
    v1 = insert(store, "c1", ("a",))
    assert store.lookup("c1")[0].f_r == 0.0 and store.lookup("c1")[0].cache.n_slots == 16
    store.touch(v1, 1.0)
    v2 = insert(store, "c1", ("a",))
    assert v1 == v2 and len(store.lookup("c1")) == 1 and store.get(v1).f_r == 1.0
    insert(store, "c1", ("b",))
    assert len(store.lookup("c1")) == 2
    assert store.lookup("nope") == []


def test_touch_inverse_cfo_and_floor():
    store = VariantStore(StoreConfig())
    vid = insert(store, "c1")
    assert store.touch(vid, 0.5) == pytest.approx(2.0)
    assert store.touch(vid, 1.0) == pytest.approx(3.0)
    assert store.touch(vid, 0.0) == pytest.approx(103.0)
    with pytest.raises(NotFoundError):
        store.touch(999, 0.5)


def test_eviction_order_and_capacity():
    store = VariantStore(StoreConfig(max_chunks=2, variants_per_chunk=2))
    vids = [insert(store, f"c{i}") for i in range(4)]
    for v, fr in zip(vids, (3.0, 0.5, 2.0, 1.0)):
        store.get(v).f_r = fr
    assert store.evict(1) == [vids[1]]
    insert(store, "c9")
    insert(store, "c10")
    assert len(store) == 4
    assert VariantStore(StoreConfig()).evict(3) == []
    with pytest.raises(ArgumentError):
        store.evict(0)


@settings(max_examples=20, deadline=None)
@given(seed=st.integers(0, 2**31 - 1))
def test_capacity_and_victim_minimality(seed):
    r = np.random.default_rng(seed)
    cfg = StoreConfig(max_chunks=3, variants_per_chunk=2)
    store = VariantStore(cfg)
    for _ in range(120):
        op = r.integers(0, 3)
        if op == 0 or len(store) == 0:
            before = {v.variant_id: (v.f_r, v.created_at) for v in store.variants()}
            vid = insert(store, f"c{r.integers(0, 6)}", (f"p{r.integers(0, 3)}",))
            after = {v.variant_id for v in store.variants()}
            gone = set(before) - after
            if gone:  # victims had the globally smallest (f_r, age)
                floor = min(before[g] for g in gone)
                survivors = [before[v] for v in after if v in before]
                assert all(s >= floor for s in survivors)
        elif op == 1:
            v = store.variants()[r.integers(0, len(store))]
            store.touch(v.variant_id, float(r.uniform(0, 1)))
        else:
            store.evict(1)
        assert len(store) <= cfg.capacity


def test_snapshot_round_trip(tmp_path):
    store = VariantStore(StoreConfig(max_chunks=4, variants_per_chunk=2))
    vids = [insert(store, f"c{i}", ("p",), n=10 + i) for i in range(3)]
    store.touch(vids[0], 0.25)
    store.snapshot(tmp_path)
    loaded = VariantStore.load_snapshot(tmp_path)
    assert len(loaded) == len(store)
    for v in store.variants():
        w = loaded.get(v.variant_id)
        assert w.prefix == v.prefix and w.f_r == pytest.approx(v.f_r)
        np.testing.assert_allclose(w.cache.keys[1], v.cache.keys[1])  # f32 wire format
        assert w.cache.n_tokens == v.cache.n_tokens
