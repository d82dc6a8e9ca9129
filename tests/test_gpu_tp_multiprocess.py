"""The production tensor-parallel data plane across real processes, on the
one GPU the test box has (reference model.py:417, :419 — the two reductions
of a layer).

Two ranks are spawned as separate processes, both on cuda:0, joined by a
``gloo`` process group (NCCL refuses two ranks on one device; gloo reduces
CUDA tensors).  Each rank builds its head/column shard of a small
Llama-shaped model through ``build_model(cfg, tp=TPContext(slices))`` and
runs the fix-up prefill with:

* the DEFAULT all-reduce (``TPContext.allreduce_`` -> ``dist.all_reduce``)
  after o_proj and down_proj, fp64 and bf16; and
* the fused peer path's cross-process plumbing (``test_ipc_peer_push_reduce
  _across_processes``): ``PeerComm.over_ipc`` exchanges CUDA-IPC handles over
  torch.distributed and maps the other process's buffers; each rank's push
  GEMM writes its fp32 tiles into the owner's slab through the mapped
  pointers, the owner reduction sums them in rank order and all-gathers,
  and the done counters advance — the production kernels of csrc/tp_peer.cu.
  On one time-sliced GPU two processes cannot spin on each other (measured:
  the concurrent schedule stalls), so the three phases are separated by host
  barriers; on an 8-GPU box the ranks run them back to back.

Both ranks must hold the unsharded model's result (oracle), and each rank's
K/V columns must be its slice of the oracle's.  Every child runs under a
deadline; a hung rank is killed (its context, and its kernels, go with it).
"""
import os
import socket
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KW = dict(n_layers=2, n_heads=8, d_model=512, d_head=64, vocab_size=512, rpe_base=500000.0, seed=3, n_kv_heads=2,
          d_ff=1024, mlp="swiglu", norm_weight=True, rms_eps=1e-5)
WORLD = 2
DEADLINE_S = 240


def _request_inputs():
    from oracle import cachecraft_oracle as O

    r = np.random.default_rng(2)
    chunks = [r.integers(0, 512, n) for n in (64, 48)]
    q = r.integers(0, 512, 16)
    masks = [r.uniform(size=c.size) < 0.25 for c in chunks]
    ocfg = O.OracleConfig(**KW)
    w = O.draw_weights(ocfg)
    lay0 = O.layout([{"tokens": c} for c in chunks], [])
    o0 = O.prefill(w, ocfg, lay0, [None] * 2)
    ocaches = [([k[s:e] for k in o0["keys"]], [v[s:e] for v in o0["values"]]) for s, e in lay0["segment_slots"]]
    return chunks, q, masks, ocaches, w, ocfg


def _rank_main(rank, port, out_dir, dtype, use_peer):
    import torch.distributed as dist

    import paper_2502_15734_b200 as cc
    from paper_2502_15734_b200 import parallel

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    try:
        torch.cuda.set_device(0)
        cfg = cc.ModelConfig(dtype=dtype, **KW)
        sl = parallel.tp_slices(cfg.n_heads, cfg.kv_heads(), cfg.ff_dim(), rank, WORLD)
        peer = parallel.PeerComm.over_ipc(rank, WORLD, cfg.d_model, 256, "cuda") if use_peer else None
        tp = parallel.TPContext(sl, peer=peer)  # no injected all-reduce: the production one
        model = cc.build_model(cfg, tp=tp)
        chunks, q, masks, ocaches, _, _ = _request_inputs()
        segs = [cc.Segment(tokens=c, cache=cc.ChunkCache(keys=k, values=v, n_tokens=c.size), recompute=m)
                for c, (k, v), m in zip(chunks, ocaches, masks)]
        calls_before = dict(cc._native.calls)
        res = cc.prefill(model, cc.build_request(segs, q), first_token=True, record_attention=False)
        torch.cuda.synchronize()
        pushed = cc._native.calls.get("cc_tp_push_gemm", 0) - calls_before.get("cc_tp_push_gemm", 0)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), hidden=res.hidden,
                 keys=np.stack([res.kv.keys[l] for l in range(KW["n_layers"])]), token=res.first_token,
                 pushed=pushed)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(out_dir, dtype, use_peer, fn=None, deadline=DEADLINE_S):
    import torch.multiprocessing as mp

    ctx = mp.start_processes(fn or _rank_main, args=(_free_port(), str(out_dir), dtype, use_peer), nprocs=WORLD,
                             join=False, start_method="spawn")
    t0 = time.time()
    try:
        while not ctx.join(timeout=5):
            if time.time() - t0 > deadline:
                phases = {f: open(os.path.join(out_dir, f)).read() for f in os.listdir(out_dir) if f.startswith("phase")}
                raise TimeoutError(f"tensor-parallel ranks did not finish in {deadline} s (phases {phases})")
    finally:
        for p in ctx.processes:
            if p.is_alive():
                p.kill()


@pytest.mark.parametrize("dtype,tol,use_peer", [("fp64", 1e-9, False), ("bf16", 2e-2, False)])
def test_two_process_tensor_parallel_matches_oracle(tmp_path, dtype, tol, use_peer):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from oracle import cachecraft_oracle as O

    _spawn(tmp_path, dtype, use_peer)
    chunks, q, masks, ocaches, w, ocfg = _request_inputs()
    lay = O.layout([{"tokens": c, "n_slots": c.size, "recompute": m} for c, m in zip(chunks, masks)], q)
    ref = O.prefill(w, ocfg, lay, ocaches)
    want_tok = O.greedy_token(w, ocfg, ref)
    out = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(WORLD)]
    for r in range(WORLD):
        h = out[r]["hidden"]
        err = np.linalg.norm(h - ref["hidden"]) / np.linalg.norm(ref["hidden"])
        assert err < tol, (r, err)
        assert int(out[r]["token"]) == want_tok
        # the fused path really ran: 2 pushes (o_proj, down_proj) per layer
        assert int(out[r]["pushed"]) == (2 * KW["n_layers"] if use_peer else 0)
    # both ranks hold identical residual streams (the sum is the same bits everywhere)
    assert np.array_equal(out[0]["hidden"], out[1]["hidden"])
    for l in range(KW["n_layers"]):
        k = np.concatenate([out[0]["keys"][l], out[1]["keys"][l]], axis=1)
        err = np.linalg.norm(k - ref["keys"][l]) / np.linalg.norm(ref["keys"][l])
        assert err < tol, (l, err)


def _ipc_rank_main(rank, port, out_dir, dtype, use_peer):
    import ctypes

    import torch.distributed as dist

    from paper_2502_15734_b200 import _native as N
    from paper_2502_15734_b200 import parallel

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    try:
        torch.cuda.set_device(0)
        d, k, M = 512, 256, 200

        def mark(phase):  # progress marker: a hang names its phase
            with open(os.path.join(out_dir, f"phase{rank}"), "w") as fh:
                fh.write(phase)

        mark("over_ipc")
        comm = parallel.PeerComm.over_ipc(rank, WORLD, d, 256, "cuda")
        mark("push")
        g = torch.Generator(device="cuda").manual_seed(100 + rank)
        A = torch.randn((M, k), generator=g, device="cuda").bfloat16()
        B = (torch.randn((d, k), generator=g, device="cuda") / k ** 0.5).bfloat16()
        s = torch.cuda.current_stream().cuda_stream
        comm.epoch += 1
        tab = comm.table()
        N.call("cc_tp_push_gemm", N.ptr(A), k, N.ptr(B), k, M, d, k, ctypes.addressof(tab), s)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's tiles are in their owners' slabs
        mark("reduce")
        N.call("cc_tp_reduce", ctypes.addressof(tab), M, d, s)
        torch.cuda.synchronize()
        dist.barrier()  # every owner has all-gathered its columns
        comm.done_target += (-(-M // 128)) * (d // 256)
        mark("wait")
        N.call("cc_tp_wait", ctypes.addressof(tab), comm.done_target, s)
        torch.cuda.synchronize()
        np.savez(os.path.join(out_dir, f"ipc{rank}.npz"), A=A.float().cpu().numpy(), B=B.float().cpu().numpy(),
                 sum=comm.local["sum"][:M].cpu().numpy(), done=comm.local["done"][:1].cpu().numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_ipc_peer_push_reduce_across_processes(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    _spawn(tmp_path, "bf16", True, fn=_ipc_rank_main, deadline=90)
    out = [np.load(os.path.join(tmp_path, f"ipc{r}.npz")) for r in range(WORLD)]
    want = sum(o["A"] @ o["B"].T for o in out)  # fp32 partials summed over the ranks
    for r in range(WORLD):
        np.testing.assert_allclose(out[r]["sum"], want, rtol=1e-3, atol=1e-3)
        assert int(out[r]["done"][0]) == (-(-200 // 128)) * (512 // 256)
    # owners reduce in rank order and all-gather: both ranks hold the same bits
    assert np.array_equal(out[0]["sum"], out[1]["sum"])
