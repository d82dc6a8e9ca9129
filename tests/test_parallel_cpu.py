"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic:
request sharding, the tensor-parallel partition (checked against the
unpartitioned oracle with a real all-reduce), and the bench's max-over-ranks
timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cachecraft_oracle as O
from paper_2502_15734_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def test_shard_requests_disjoint_and_complete():
    r = np.random.default_rng(0)
    recs = [list(r.integers(0, 50, 5)) for _ in range(200)]
    for policy in ("affinity", "round_robin"):
        parts = [parallel.shard_requests(recs, k, 4, policy) for k in range(4)]
        assert sum(len(p) for p in parts) == len(recs)
        ids = [id(x) for p in parts for x in p]
        assert len(set(ids)) == len(recs)
    # affinity: requests with the same leading chunk meet on the same rank
    owners = {}
    for rec in recs:
        o = parallel.request_owner(rec, 4)
        assert owners.setdefault(rec[0], o) == o


def test_tp_slices_cover_heads_and_columns():
    H, Hkv, ff, w = 64, 8, 28672, 8
    sl = [parallel.tp_slices(H, Hkv, ff, r, w) for r in range(w)]
    assert [s.q_heads for s in sl] == [(8 * r, 8) for r in range(w)]
    assert [s.kv_heads for s in sl] == [(r, 1) for r in range(w)]
    assert sum(s.ff[1] for s in sl) == ff
    # every rank's q heads read only its own kv head (GQA groups intact)
    for s in sl:
        assert s.q_heads[0] // (H // Hkv) == s.kv_heads[0]
    with pytest.raises(Exception):
        parallel.tp_slices(64, 8, 28672, 0, 3)


def _tp_worker(rank, world, kw, chunks, question, masks, out_dir):
    cfg = O.OracleConfig(**kw)
    w = O.draw_weights(cfg)
    lay0 = O.layout([{"tokens": c} for c in chunks], [])
    r0 = O.prefill(w, cfg, lay0, [None] * len(chunks))
    caches = [([k[s:e] for k in r0["keys"]], [v[s:e] for v in r0["values"]]) for s, e in lay0["segment_slots"]]
    sl = parallel.tp_slices(cfg.n_heads, cfg.hkv, cfg.ff, rank, world)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    lay = O.layout([{"tokens": c, "n_slots": c.size, "recompute": m} for c, m in zip(chunks, masks)], question)
    tp = {"q": sl.q_cols(cfg.dh), "kv": sl.kv_cols(cfg.dh), "ff": sl.ff_cols(), "allreduce": allreduce}
    res = O.prefill(w, cfg, lay, caches, tp=tp)
    np.save(os.path.join(out_dir, f"hidden{rank}.npy"), res["hidden"])
    np.save(os.path.join(out_dir, f"k0_{rank}.npy"), res["keys"][1])


@pytest.mark.parametrize("kw", [
    dict(n_layers=2, n_heads=4, d_model=64),  # reference architecture (MHA, GELU)
    dict(n_layers=2, n_heads=8, d_model=128, n_kv_heads=2, d_ff=256, mlp="swiglu", norm_weight=True,
         rpe_base=500000.0, rms_eps=1e-5),  # Llama-shaped (GQA 4:1, SwiGLU)
])
def test_tensor_parallel_partition_matches_full_model(tmp_path, kw):
    r = np.random.default_rng(5)
    chunks = [r.integers(0, 256, n) for n in (24, 16)]
    question = r.integers(0, 256, 8)
    masks = [r.uniform(size=c.size) < 0.3 for c in chunks]
    _run(2, _tp_worker, kw, chunks, question, masks, str(tmp_path))
    cfg = O.OracleConfig(**kw)
    w = O.draw_weights(cfg)
    lay0 = O.layout([{"tokens": c} for c in chunks], [])
    r0 = O.prefill(w, cfg, lay0, [None] * 2)
    caches = [([k[s:e] for k in r0["keys"]], [v[s:e] for v in r0["values"]]) for s, e in lay0["segment_slots"]]
    lay = O.layout([{"tokens": c, "n_slots": c.size, "recompute": m} for c, m in zip(chunks, masks)], question)
    full = O.prefill(w, cfg, lay, caches)
    for rank in range(2):
        h = np.load(tmp_path / f"hidden{rank}.npy")
        np.testing.assert_allclose(h, full["hidden"], atol=1e-10)  # hidden is replicated after each all-reduce
    # each rank holds its kv-head slice of the repaired KV
    k_parts = [np.load(tmp_path / f"k0_{rank}.npy") for rank in range(2)]
    np.testing.assert_allclose(np.concatenate(k_parts, axis=1), full["keys"][1], atol=1e-10)


def _timing_worker(rank, world):
    import bench

    assert bench.allreduce_max(1.0 + rank, world) == float(world)


def test_bench_timing_is_max_over_ranks():
    _run(2, _timing_worker)


def test_peer_table_matches_c_layout():
    """parallel._Peers mirrors cc_tp_peers (include/cachecraft_b200.h):
    4 x 8 pointers then rank, world, slice, m_cap, epoch (int32)."""
    import ctypes

    from paper_2502_15734_b200.parallel import _Peers

    assert ctypes.sizeof(_Peers) == 4 * 8 * 8 + 5 * 4 + 4  # 8-byte aligned tail
    assert _Peers.rank.offset == 256 and _Peers.epoch.offset == 272
