"""Tensor-parallel engine on one B200: two TP ranks (separate shard models
and CUDA streams) run concurrently in threads; their all-reduce is a
barrier + device sum.  The composed result must equal the unsharded model
(and the oracle), i.e. the sharded kernels + the two all-reduces per layer
reproduce model.py:348-442."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from ccb_helpers import record_measurement  # noqa: E402
from oracle import cachecraft_oracle as O  # noqa: E402


class ThreadGroup:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.buf = [None] * world

    def allreduce_for(self, rank):
        def ar(t):
            torch.cuda.current_stream().synchronize()
            self.buf[rank] = t
            self.bar.wait()
            if rank == 0:
                total = sum(b.clone() for b in self.buf)
                for b in self.buf:
                    b.copy_(total)
                torch.cuda.synchronize()
            self.bar.wait()
            return t
        return ar


@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-9), ("bf16", 1.2e-2)])  # bf16: 3x measured (4.0e-3)
def test_two_rank_tensor_parallel_matches_unsharded(dtype, tol):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2502_15734_b200 as cc
    from paper_2502_15734_b200 import parallel

    kw = dict(n_layers=2, n_heads=8, d_model=512, d_head=64, vocab_size=512, rpe_base=500000.0, seed=3,
              n_kv_heads=2, d_ff=1024, mlp="swiglu", norm_weight=True, rms_eps=1e-5)
    cfg = cc.ModelConfig(dtype=dtype, **kw)
    r = np.random.default_rng(2)
    chunks = [r.integers(0, 512, n) for n in (64, 48)]
    q = r.integers(0, 512, 16)
    masks = [r.uniform(size=c.size) < 0.25 for c in chunks]
    # creation caches from the oracle (full width); each rank uploads its kv slice
    ocfg = O.OracleConfig(**kw)
    w = O.draw_weights(ocfg)
    lay0 = O.layout([{"tokens": c} for c in chunks], [])
    o0 = O.prefill(w, ocfg, lay0, [None] * 2)
    ocaches = [([k[s:e] for k in o0["keys"]], [v[s:e] for v in o0["values"]]) for s, e in lay0["segment_slots"]]
    lay = O.layout([{"tokens": c, "n_slots": c.size, "recompute": m} for c, m in zip(chunks, masks)], q)
    ref = O.prefill(w, ocfg, lay, ocaches)

    group = ThreadGroup(2)
    results = [None, None]
    errors = []

    def rank_main(rank):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sl = parallel.tp_slices(cfg.n_heads, cfg.kv_heads(), cfg.ff_dim(), rank, 2)
                tp = parallel.TPContext(sl, allreduce=group.allreduce_for(rank))
                model = cc.build_model(cfg, tp=tp)
                segs = [cc.Segment(tokens=c, cache=cc.ChunkCache(keys=k, values=v, n_tokens=c.size), recompute=m)
                        for c, (k, v), m in zip(chunks, ocaches, masks)]
                res = cc.prefill(model, cc.build_request(segs, q), first_token=True, record_attention=False)
                stream.synchronize()
                results[rank] = (res.hidden, [res.kv.keys[l] for l in range(2)], res.first_token)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            group.bar.abort()

    th = [threading.Thread(target=rank_main, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    errs = {"hidden": 0.0, "keys": 0.0}
    for rank in range(2):
        h, keys, tok = results[rank]
        err = np.linalg.norm(h - ref["hidden"]) / np.linalg.norm(ref["hidden"])
        errs["hidden"] = max(errs["hidden"], float(err))
        assert err < tol, (rank, err)
        assert tok == O.greedy_token(w, ocfg, ref)
    for l in range(2):
        k = np.concatenate([results[0][1][l], results[1][1][l]], axis=1)
        err = np.linalg.norm(k - ref["keys"][l]) / np.linalg.norm(ref["keys"][l])
        errs["keys"] = max(errs["keys"], float(err))
        assert err < tol
    record_measurement("tp2_in_process", {"dtype": dtype, **errs})


def test_peer_push_gemm_and_reduction_two_ranks():
    """Fused TP reduction (csrc/tp_peer.cu) with two ranks' buffers on one
    GPU, driven from one thread (no cross-rank spin can wait on an unlaunched
    peer): each rank's GEMM pushes its fp32 tiles into the column owner's
    slab, the owners reduce in rank order and all-gather; both ranks must hold
    the same bits, equal to the fp32 sum of the partials."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import ctypes

    from paper_2502_15734_b200 import _native as N
    from paper_2502_15734_b200 import parallel

    N.lib()
    world, d, k, M = 2, 512, 256, 200
    comms = parallel.PeerComm.in_process(world, d, 256, "cuda")
    g = torch.Generator(device="cuda").manual_seed(11)
    A = [torch.randn((M, k), generator=g, device="cuda").bfloat16() for _ in range(world)]
    B = [(torch.randn((d, k), generator=g, device="cuda") / k ** 0.5).bfloat16() for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    for step in range(2):  # two calls: epochs and the monotonic done counter advance
        tabs = []
        for r in range(world):
            comms[r].epoch += 1
            tabs.append(comms[r].table())
        torch.cuda.synchronize()
        for r in range(world):
            N.call("cc_tp_push_gemm", N.ptr(A[r]), k, N.ptr(B[r]), k, M, d, k, ctypes.addressof(tabs[r]),
                   streams[r].cuda_stream)
        for r in range(world):
            N.call("cc_tp_reduce", ctypes.addressof(tabs[r]), M, d, streams[r].cuda_stream)
        for r in range(world):
            comms[r].done_target += (-(-M // 128)) * (d // 256)
            N.call("cc_tp_wait", ctypes.addressof(tabs[r]), comms[r].done_target, streams[r].cuda_stream)
        torch.cuda.synchronize()
        ref = sum(a.float() @ b.float().T for a, b in zip(A, B))
        s0 = comms[0].local["sum"][:M]
        s1 = comms[1].local["sum"][:M]
        assert torch.equal(s0, s1)
        torch.testing.assert_close(s0, ref, atol=1e-3, rtol=1e-3)
        A = [a.flip(0).contiguous() for a in A]
