"""build_plan decisions (HIT/MISS, min-CFO variant, CFO, K9 recompute sets)
bit-exact against the reference fixture (planner.py:132-179)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from ccb_helpers import load_json  # noqa: E402


def test_build_plan_matches_reference_fixture():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2502_15734_b200 as cc

    g = load_json("plan.json")
    chunks = [np.asarray(c, dtype=np.int64) for c in g["chunks"]]
    ids = [cc.chunk_hash(c) for c in chunks]
    # rebuild the generator's store by replaying its random stream (tests/golden/make_golden.py:gen_plan)
    store2 = cc.VariantStore(cc.StoreConfig(max_chunks=3, variants_per_chunk=3))
    r = np.random.default_rng(31)
    # regenerate the generator's random stream to recover the touch cfo values
    for c in range(5):
        r.integers(0, 256, int((8, 10, 16, 24, 9)[c]))
    for rep, ins in enumerate(g["inserts"]):
        ci = int(r.integers(0, 5))
        m = int(r.integers(0, 4))
        pool = [x for x in ids if x != ids[ci]] + ["zz", "yy"]
        pre = list(r.choice(pool, size=m, replace=False))
        w = [float(x) for x in r.uniform(0, 1, m)]
        n = chunks[ci].size
        ts = r.standard_normal(n)
        ts[r.integers(0, n, 2)] = 0.25
        cci = float(r.uniform(0.5, 1.0))
        vid = store2.insert(ids[ci], prefix=cc.PrefixContext(chunk_ids=tuple(pre), weights=tuple(w)), a_bar=0.1,
                            b_bar=0.1, cci=cci, token_scores=ts,
                            cache=cc.ChunkCache(keys=[np.zeros((n, 4))], values=[np.zeros((n, 4))], n_tokens=n))
        assert vid == ins["vid"] and ci == ins["chunk"]
        if rep % 3 == 2:
            fr = store2.touch(vid, float(r.uniform(0, 1)))
            assert fr == ins["touched_fr"]
    assert [v.variant_id for v in store2.variants()] == g["live"]
    assert store2.census() == g["census"]
    for want in g["plans"]:
        r.permutation(5)  # keep the stream aligned with the generator
        r.integers(2, 6)
        r.choice([0.35, 1.0, 3.0])
        r.integers(0, 256, 4)
        plan = cc.build_plan([chunks[i] for i in want["order"]], np.zeros(4, np.int64), store2, want["alpha"])
        got = [{"status": cp.status, "variant_id": cp.variant_id, "cfo": cp.cfo,
                "recompute": [] if cp.recompute is None else [int(i) for i in cp.recompute]} for cp in plan.chunks]
        assert got == want["chunks"]
