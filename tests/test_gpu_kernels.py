"""Kernel-level parity on the B200 (through the C ABI): each CUDA kernel
against the oracle / a plain torch fp32 reference of the same op."""
import json
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from ccb_helpers import golden_path, load_json  # noqa: E402

from oracle import cachecraft_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def N():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2502_15734_b200 import _native

    _native.lib()
    return _native


def test_rope_apply_matches_reference_fixture(N):
    import paper_2502_15734_b200 as cc

    g = np.load(golden_path("rope.npz"))
    x, pos = g["x"], g["pos"]
    np.testing.assert_allclose(cc.apply_rpe(x, pos), g["apply_full"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(cc.apply_rpe(x, pos, d_head=8), g["apply_h8"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(cc.remove_rpe(x, pos, d_head=8), g["remove_h8"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(cc.apply_rpe(x, pos, base=500000.0, d_head=16), g["apply_h16_b5e5"], atol=1e-12)
    np.testing.assert_array_equal(cc.apply_rpe(x[:3], np.zeros(3)), x[:3])  # position 0 is identity


def test_topk_select_bit_exact_on_reference_vectors(N):
    import paper_2502_15734_b200 as cc

    for case in load_json("select.json"):
        assert cc.select_tokens(case["scores"], case["cfo"]).tolist() == case["selected"]


def test_topk_select_random_ties_and_batches(N):
    from paper_2502_15734_b200.planner import recompute_count, select_tokens_batched

    r = np.random.default_rng(0)
    scores, counts = [], []
    for n in (1, 3, 16, 100, 128, 512, 1000, 1024, 4096):
        s = np.round(r.standard_normal(n), 1)  # heavy ties
        c = float(r.uniform())
        scores.append(s)
        counts.append(recompute_count(n, c))
    got = select_tokens_batched(scores, counts)
    for s, k, gsel in zip(scores, counts, got):
        want = np.sort(np.argsort(-s, kind="stable")[:k])
        np.testing.assert_array_equal(gsel, want)


def _gemm(N, A, B, epi, dtype, impl, C=None):
    M, K = A.shape
    Nn = B.shape[0]
    if C is None:
        n_out = Nn // 2 if epi == N.EPI_SWIGLU else Nn
        C = torch.zeros((M, n_out), dtype=A.dtype, device="cuda")
    N.call("cc_gemm", N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, epi, dtype, impl, N.stream_ptr())
    torch.cuda.synchronize()
    return C


@pytest.mark.parametrize("M", [1, 77, 128, 130, 802])
@pytest.mark.parametrize("NK", [(256, 64), (768, 256), (512, 4096), (6144, 256), (384, 512)])
def test_gemm_tcgen05_store_matches_fp32_reference(N, M, NK):
    Nn, K = NK
    g = torch.Generator(device="cuda").manual_seed(M * 7 + Nn)
    A = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    B = (torch.randn((Nn, K), generator=g, device="cuda") / math.sqrt(K)).bfloat16()
    ref = A.float() @ B.float().T
    tc = _gemm(N, A, B, N.EPI_STORE, N.BF16, 1)
    simt = _gemm(N, A, B, N.EPI_STORE, N.BF16, 2)
    torch.testing.assert_close(tc.float(), ref, atol=2e-2, rtol=1e-2)
    torch.testing.assert_close(simt.float(), ref, atol=2e-2, rtol=1e-2)


@pytest.mark.parametrize("epi", ["resid", "swiglu", "gelu"])
def test_gemm_tcgen05_epilogues(N, epi):
    M, Nn, K = 300, 1024, 512
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    B = (torch.randn((Nn, K), generator=g, device="cuda") / math.sqrt(K)).bfloat16()
    acc = A.float() @ B.float().T
    if epi == "resid":
        H0 = torch.randn((M, Nn), generator=g, device="cuda")
        H = H0.clone()
        _gemm(N, A, B, N.EPI_RESID_ADD, N.BF16, 1, C=H)
        torch.testing.assert_close(H, H0 + acc, atol=1e-3, rtol=1e-3)
    elif epi == "swiglu":
        out = _gemm(N, A, B, N.EPI_SWIGLU, N.BF16, 1)
        a4 = acc.reshape(M, Nn // 128, 2, 64)
        ref = (torch.nn.functional.silu(a4[:, :, 0]) * a4[:, :, 1]).reshape(M, Nn // 2)
        torch.testing.assert_close(out.float(), ref, atol=2e-2, rtol=2e-2)
        out2 = _gemm(N, A, B, N.EPI_SWIGLU, N.BF16, 2)
        torch.testing.assert_close(out2.float(), ref, atol=2e-2, rtol=2e-2)
    else:
        out = _gemm(N, A, B, N.EPI_GELU, N.BF16, 1)
        ref = torch.nn.functional.gelu(acc, approximate="tanh")
        torch.testing.assert_close(out.float(), ref, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("bn", [224, 160])
@pytest.mark.parametrize("epi", ["store", "resid"])
def test_gemm_ragged_tile_width(N, bn, epi, monkeypatch):
    """Tile widths that do not divide N (ragged last tile, TMA zero fill,
    masked epilogue) match the fp32 reference."""
    import subprocess
    import sys

    code = f"""
import torch, sys
sys.path.insert(0, '.')
from paper_2502_15734_b200 import _native as N
M, Nn, K = 802, 4096, 1024
g = torch.Generator(device='cuda').manual_seed(2)
A = torch.randn((M, K), generator=g, device='cuda').bfloat16()
B = (torch.randn((Nn, K), generator=g, device='cuda') / 32).bfloat16()
acc = A.float() @ B.float().T
if '{epi}' == 'resid':
    C = torch.ones((M, Nn), device='cuda'); ref = acc + 1
    N.call('cc_gemm', N.ptr(A), K, N.ptr(B), K, N.ptr(C), Nn, M, Nn, K, N.EPI_RESID_ADD, N.BF16, 1, N.stream_ptr())
else:
    C = torch.empty((M, Nn), device='cuda', dtype=torch.bfloat16); ref = acc
    N.call('cc_gemm', N.ptr(A), K, N.ptr(B), K, N.ptr(C), Nn, M, Nn, K, N.EPI_STORE, N.BF16, 1, N.stream_ptr())
torch.testing.assert_close(C.float(), ref, atol=2e-2, rtol=2e-2)
print('ok')
"""
    env = dict(__import__("os").environ, CCB_GEMM_FORCE=f"{bn},0")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("bnr", [208, 144, 256])
@pytest.mark.parametrize("epi", ["store", "resid", "gelu"])
def test_gemm_swap_ab(N, bnr, epi):
    """Swap-AB tiles (weights as the MMA M side, activation rows as N with a
    ragged last row tile) match the fp32 reference for every epilogue."""
    import subprocess
    import sys

    code = f"""
import torch, sys
sys.path.insert(0, '.')
from paper_2502_15734_b200 import _native as N
M, Nn, K = 802, 1536, 1024
g = torch.Generator(device='cuda').manual_seed(4)
A = torch.randn((M, K), generator=g, device='cuda').bfloat16()
B = (torch.randn((Nn, K), generator=g, device='cuda') / 32).bfloat16()
acc = A.float() @ B.float().T
epi = '{epi}'
if epi == 'resid':
    C = torch.ones((M, Nn), device='cuda'); ref = acc + 1; code = N.EPI_RESID_ADD
elif epi == 'swiglu':
    C = torch.empty((M, Nn // 2), device='cuda', dtype=torch.bfloat16); code = N.EPI_SWIGLU
    a4 = acc.reshape(M, Nn // 128, 2, 64); ref = (torch.nn.functional.silu(a4[:, :, 0]) * a4[:, :, 1]).reshape(M, Nn // 2)
else:
    C = torch.empty((M, Nn), device='cuda', dtype=torch.bfloat16)
    code = N.EPI_GELU if epi == 'gelu' else N.EPI_STORE
    ref = torch.nn.functional.gelu(acc, approximate='tanh') if epi == 'gelu' else acc
N.call('cc_gemm', N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, code, N.BF16, 1, N.stream_ptr())
torch.testing.assert_close(C.float(), ref, atol=2e-2, rtol=2e-2)
print('ok')
"""
    env = dict(__import__("os").environ, CCB_GEMM_FORCE=f"{bnr},2")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("M", [802, 300, 37])
@pytest.mark.parametrize("epi", ["store", "resid", "swiglu", "gelu"])
def test_gemm_cta_pair_unit_table(N, M, epi):
    """CTA-pair (cta_group::2) swap-AB GEMM with the host-planned unit table
    and TMA-store / TMA-reduce-add epilogues: matches the fp32 reference and
    is bit-identical to the 1-CTA data-parallel tiling."""
    import subprocess
    import sys

    code = f"""
import math, torch, sys
sys.path.insert(0, '.')
from paper_2502_15734_b200 import _native as N
M, Nn, K = {M}, 1536, 1024
g = torch.Generator(device='cuda').manual_seed(6)
A = torch.randn((M, K), generator=g, device='cuda').bfloat16()
B = (torch.randn((Nn, K), generator=g, device='cuda') / 32).bfloat16()
acc = A.float() @ B.float().T
epi = '{epi}'
code = dict(store=N.EPI_STORE, resid=N.EPI_RESID_ADD, swiglu=N.EPI_SWIGLU, gelu=N.EPI_GELU)[epi]
if epi == 'resid':
    C = torch.ones((M, Nn), device='cuda'); ref = acc + 1
elif epi == 'swiglu':
    C = torch.empty((M, Nn // 2), device='cuda', dtype=torch.bfloat16)
    a4 = acc.reshape(M, Nn // 128, 2, 64); ref = (torch.nn.functional.silu(a4[:, :, 0]) * a4[:, :, 1]).reshape(M, Nn // 2)
else:
    C = torch.empty((M, Nn), device='cuda', dtype=torch.bfloat16)
    ref = torch.nn.functional.gelu(acc, approximate='tanh') if epi == 'gelu' else acc
N.call('cc_gemm', N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, code, N.BF16, 4, N.stream_ptr())
torch.testing.assert_close(C.float(), ref, atol=2e-2, rtol=2e-2)
torch.save(C.cpu(), sys.argv[1])
print('ok')
"""
    outs = []
    for i, force in enumerate(["0,4", "256,0"]):
        path = f"/tmp/_pair_{epi}_{M}_{i}.pt"
        env = dict(__import__("os").environ, CCB_GEMM_FORCE=force)
        out = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True, env=env, timeout=300)
        assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
        outs.append(torch.load(path))
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("M,S", [(96, 2), (290, 3), (290, 4), (545, 6)])
@pytest.mark.parametrize("epi", ["store", "resid", "swiglu", "gelu"])
def test_gemm_cta_pair_k_split(N, M, S, epi):
    """CTA-pair units with the K dimension split into S slices (small M):
    each slice's CTA parks an fp32 partial, the last to finish a unit sums
    them in slice order and runs the epilogue.  Matches the fp32 reference,
    equals the unsplit pair plan within fp32 re-association, and is
    bit-identical from run to run (whichever CTA finishes last)."""
    import subprocess
    import sys

    code = f"""
import torch, sys
sys.path.insert(0, '.')
from paper_2502_15734_b200 import _native as N
M, Nn, K = {M}, 1536, 4096
g = torch.Generator(device='cuda').manual_seed(7)
A = torch.randn((M, K), generator=g, device='cuda').bfloat16()
B = (torch.randn((Nn, K), generator=g, device='cuda') / 64).bfloat16()
acc = A.float() @ B.float().T
epi = '{epi}'
code = dict(store=N.EPI_STORE, resid=N.EPI_RESID_ADD, swiglu=N.EPI_SWIGLU, gelu=N.EPI_GELU)[epi]
def run():
    if epi == 'resid':
        C = torch.ones((M, Nn), device='cuda')
    elif epi == 'swiglu':
        C = torch.empty((M, Nn // 2), device='cuda', dtype=torch.bfloat16)
    else:
        C = torch.empty((M, Nn), device='cuda', dtype=torch.bfloat16)
    N.call('cc_gemm', N.ptr(A), K, N.ptr(B), K, N.ptr(C), C.shape[1], M, Nn, K, code, N.BF16, 1, N.stream_ptr())
    torch.cuda.synchronize()
    return C
if epi == 'resid':
    ref = acc + 1
elif epi == 'swiglu':
    a4 = acc.reshape(M, Nn // 128, 2, 64); ref = (torch.nn.functional.silu(a4[:, :, 0]) * a4[:, :, 1]).reshape(M, Nn // 2)
else:
    ref = torch.nn.functional.gelu(acc, approximate='tanh') if epi == 'gelu' else acc
outs = [run() for _ in range(3)]
torch.testing.assert_close(outs[0].float(), ref, atol=2e-2, rtol=2e-2)
assert all(torch.equal(outs[0], o) for o in outs[1:])
torch.save(outs[0].cpu(), sys.argv[1])
print('ok')
"""
    outs = []
    for i, force in enumerate([f"{S},5", "0,4"]):
        path = f"/tmp/_ksplit_{epi}_{M}_{S}_{i}.pt"
        env = dict(__import__("os").environ, CCB_GEMM_FORCE=force, CCB_SW_DEBUG="1")
        out = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True, env=env, timeout=300)
        assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
        if i == 0:
            assert f"slices={S}" in out.stderr, out.stderr[-500:]
        outs.append(torch.load(path).float())
    # slices re-associate the fp32 sum: the unsplit result within a bf16 ulp or two
    torch.testing.assert_close(outs[0], outs[1], atol=1e-2, rtol=1e-2)


def test_gemm_k_split_concurrent_streams(N):
    """K-split units on several CUDA streams at once (the serving mode runs
    requests on separate streams): each stream has its own partial workspace
    and tickets, so concurrent launches give the single-stream bits."""
    M, Nn, K = 96, 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(11)
    A = [torch.randn((M, K), generator=g, device="cuda").bfloat16() for _ in range(4)]
    B = (torch.randn((Nn, K), generator=g, device="cuda") / 64).bfloat16()

    def run(i, stream):
        C = torch.ones((M, Nn), device="cuda")
        stream.wait_stream(torch.cuda.current_stream())  # (C is filled on the current stream)
        N.call("cc_gemm", N.ptr(A[i]), K, N.ptr(B), K, N.ptr(C), Nn, M, Nn, K, N.EPI_RESID_ADD, N.BF16, 0,
               N.stream_ptr(stream))
        return C

    base = []
    for i in range(4):
        base.append(run(i, torch.cuda.current_stream()))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(4)]
    for rep in range(3):
        outs = [run(i, streams[i]) for i in range(4)]
        torch.cuda.synchronize()
        for i in range(4):
            assert torch.equal(outs[i], base[i]), (rep, i)
    ref = A[0].float() @ B.float().T + 1
    torch.testing.assert_close(base[0], ref, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("Nn", [512, 6144, 1536])
def test_gemm_tcgen05_m_invariance(N, Nn):
    """A row's result does not depend on how many rows are active (also when
    the tile width chosen for the two M differs)."""
    K = 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn((5152, K), generator=g, device="cuda").bfloat16()
    B = (torch.randn((Nn, K), generator=g, device="cuda") / 32).bfloat16()
    full = _gemm(N, A, B, N.EPI_STORE, N.BF16, 4)  # impl 4: tcgen05 without split-K
    part = _gemm(N, A[:37].contiguous(), B, N.EPI_STORE, N.BF16, 4)
    assert torch.equal(full[:37], part)


@pytest.mark.parametrize("M", [32, 802])
@pytest.mark.parametrize("epi", ["store", "resid", "swiglu", "gelu"])
def test_gemm_split_k_deterministic(N, M, epi):
    """Split-K with in-order fix-ups: matches the fp32 reference and is
    bit-reproducible run to run."""
    Nn, K = (4096, 14336) if epi == "resid" else (2048, 4096)
    g = torch.Generator(device="cuda").manual_seed(M)
    A = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    B = (torch.randn((Nn, K), generator=g, device="cuda") / math.sqrt(K)).bfloat16()
    acc = A.float() @ B.float().T
    code = {"store": N.EPI_STORE, "resid": N.EPI_RESID_ADD, "swiglu": N.EPI_SWIGLU, "gelu": N.EPI_GELU}[epi]
    outs = []
    for _ in range(2):
        if epi == "resid":
            H = torch.ones((M, Nn), device="cuda")
            _gemm(N, A, B, code, N.BF16, 1, C=H)
            outs.append(H)
        else:
            outs.append(_gemm(N, A, B, code, N.BF16, 1))
    assert torch.equal(outs[0], outs[1])
    if epi == "resid":
        ref = acc + 1.0
        torch.testing.assert_close(outs[0], ref, atol=1e-3, rtol=1e-3)
    elif epi == "swiglu":
        a4 = acc.reshape(M, Nn // 128, 2, 64)
        ref = (torch.nn.functional.silu(a4[:, :, 0]) * a4[:, :, 1]).reshape(M, Nn // 2)
        torch.testing.assert_close(outs[0].float(), ref, atol=2e-2, rtol=2e-2)
    elif epi == "gelu":
        torch.testing.assert_close(outs[0].float(), torch.nn.functional.gelu(acc, approximate="tanh"), atol=2e-2,
                                   rtol=2e-2)
    else:
        torch.testing.assert_close(outs[0].float(), acc, atol=2e-2, rtol=1e-2)


def _attn_ref(q, k, v, q_slot, pad, Hq, Hkv):
    """plain torch fp32 reference of model.py:406-416 for scattered rows"""
    n = k.shape[0]
    dh = q.shape[-1]
    G = Hq // Hkv
    kk = k.float().repeat_interleave(G, dim=1)  # [n, Hq, dh]
    vv = v.float().repeat_interleave(G, dim=1)
    s = torch.einsum("qhd,khd->hqk", q.float(), kk) / math.sqrt(dh)
    j = torch.arange(n, device=q.device)
    ok = (j[None, :] <= q_slot[:, None].long()) & (pad[None, :] == 0)
    s = s.masked_fill(~ok[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqk,khd->qhd", p, vv).reshape(q.shape[0], Hq * dh), torch.logsumexp(s, dim=-1).T


@pytest.mark.parametrize("ext", ["0", "1"])
@pytest.mark.parametrize("n_rows,n", [(32, 5152), (150, 2100), (300, 5152)])
def test_attention_key_part_merge_modes(N, ext, n_rows, n):
    """The ping-pong kernel's key parts merged by the last part (CCB_ATTN_EXT=0)
    or by the separate attn_pp_merge kernel (=1, up to 16 parts; the default
    for <= 16 items): both match torch fp32 and are deterministic."""
    import subprocess
    import sys

    code = f"""
import math, sys, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_2502_15734_b200 import _native as N
from test_gpu_kernels import _attn_ref
Hq, Hkv, dh, n = 32, 8, 128, {n}
g = torch.Generator(device='cuda').manual_seed(3)
rows = torch.sort(torch.randperm(n, generator=g, device='cuda')[:{n_rows}]).values.int()
rows[-1] = n - 1
rows = torch.unique(rows).int().contiguous()
q = torch.randn((rows.numel(), Hq, dh), generator=g, device='cuda').bfloat16()
k = torch.randn((n, Hkv, dh), generator=g, device='cuda').bfloat16()
v = torch.randn((n, Hkv, dh), generator=g, device='cuda').bfloat16()
pad = torch.zeros(n, dtype=torch.uint8, device='cuda')
pad[40:52] = 1
rows = rows[pad[rows.long()] == 0].contiguous()
q = q[: rows.numel()].contiguous()
outs = []
for _ in range(2):
    ctx = torch.zeros((rows.numel(), Hq * dh), dtype=torch.bfloat16, device='cuda')
    lse = torch.zeros((rows.numel(), Hq), dtype=torch.float32, device='cuda')
    N.call('cc_attention', N.ptr(q), N.ptr(k), N.ptr(v), N.ptr(rows), N.ptr(pad), N.ptr(ctx), N.ptr(lse),
           rows.numel(), n, Hq, Hkv, dh, N.BF16, 1, N.stream_ptr())
    torch.cuda.synchronize()
    outs.append((ctx, lse))
ref, ref_lse = _attn_ref(q, k, v, rows, pad, Hq, Hkv)
torch.testing.assert_close(outs[0][0].float(), ref, atol=3e-2, rtol=3e-2)
torch.testing.assert_close(outs[0][1], ref_lse, atol=2e-3, rtol=1e-3)
assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
print('ok')
"""
    env = dict(__import__("os").environ, CCB_ATTN_EXT=ext)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("Hq,Hkv,dh,n", [(32, 8, 128, 700), (4, 4, 64, 700), (8, 1, 128, 700), (16, 2, 64, 700),
                                          (32, 8, 128, 2100), (64, 8, 128, 300), (32, 8, 128, 5152)])
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_attention_scattered_rows(N, Hq, Hkv, dh, n, variant):
    """impl 1 = tcgen05/TMEM kernel in each tile shape (variant: 128- or
    64-key tiles, one or two softmax warpgroups; key ranges split for the
    long row tiles when the grid is small, merged in fixed order),
    2 = SIMT reference."""
    import ctypes

    N.lib().cc_debug_attn_variant.argtypes = [ctypes.c_int]
    N.lib().cc_debug_attn_variant(variant)
    g = torch.Generator(device="cuda").manual_seed(Hq + dh)
    rows = torch.sort(torch.randperm(n, generator=g, device="cuda")[:150]).values.int()
    q = torch.randn((rows.numel(), Hq, dh), generator=g, device="cuda").bfloat16()
    k = torch.randn((n, Hkv, dh), generator=g, device="cuda").bfloat16()
    v = torch.randn((n, Hkv, dh), generator=g, device="cuda").bfloat16()
    pad = torch.zeros(n, dtype=torch.uint8, device="cuda")
    pad[100:112] = 1
    pad[400:405] = 1
    rows = rows[pad[rows.long()] == 0].contiguous()
    q = q[: rows.numel()].contiguous()
    ctx = torch.empty((rows.numel(), Hq * dh), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((rows.numel(), Hq), dtype=torch.float32, device="cuda")
    for impl in (1, 2):
        ctx.zero_()
        N.call("cc_attention", N.ptr(q), N.ptr(k), N.ptr(v), N.ptr(rows), N.ptr(pad), N.ptr(ctx), N.ptr(lse),
               rows.numel(), n, Hq, Hkv, dh, N.BF16, impl, N.stream_ptr())
        torch.cuda.synchronize()
        ref, ref_lse = _attn_ref(q, k, v, rows, pad, Hq, Hkv)
        torch.testing.assert_close(ctx.float(), ref, atol=3e-2, rtol=3e-2)
        torch.testing.assert_close(lse, ref_lse, atol=2e-3, rtol=1e-3)
        if impl == 1:  # deterministic (split merge order fixed)
            ctx2 = torch.empty_like(ctx)
            N.call("cc_attention", N.ptr(q), N.ptr(k), N.ptr(v), N.ptr(rows), N.ptr(pad), N.ptr(ctx2), N.ptr(lse),
                   rows.numel(), n, Hq, Hkv, dh, N.BF16, impl, N.stream_ptr())
            assert torch.equal(ctx, ctx2)
    N.lib().cc_debug_attn_variant(-1)


def test_gather_rope_matches_torch(N):
    """K1 against a torch reference: copy position-free rows, rotate keys."""
    L, kvw, dh = 3, 256, 128
    nb_pool = 12
    pool = torch.randn((L, nb_pool, 2, 16, kvw), device="cuda").bfloat16()
    n = 70
    items = np.array([(3, 0, 16, 0), (7, 16, 16, 0), (1, 32, 10, 0), (5, 50, 16, 0)], dtype=np.int32)
    slot_pos = torch.arange(n, dtype=torch.int32, device="cuda") + 5
    active = torch.zeros(n, dtype=torch.int32, device="cuda")
    active[20] = 2  # slot 20 recomputed through layer 1: skipped at layers 0, 1
    half = dh // 2
    inv = torch.from_numpy(500000.0 ** (-2.0 * np.arange(half) / dh)).cuda()
    tab = torch.empty((256, half, 2), dtype=torch.float32, device="cuda")
    N.call("cc_rope_table", N.ptr(tab), N.ptr(inv), 256, half, N.BF16, N.stream_ptr())
    kv_k = torch.zeros((L, n, kvw), dtype=torch.bfloat16, device="cuda")
    kv_v = torch.zeros_like(kv_k)
    k_rot = torch.zeros_like(kv_k)
    it = torch.from_numpy(items.reshape(-1)).cuda()
    N.call("cc_gather_rope_kv", N.ptr(pool), pool.stride(0), pool.stride(1), N.ptr(it), len(items), 0, L,
           N.ptr(slot_pos), N.ptr(active), N.ptr(tab), N.ptr(kv_k), N.ptr(kv_v), N.ptr(k_rot), n * kvw, kvw, dh,
           N.BF16, N.stream_ptr())
    torch.cuda.synchronize()
    for (blk, dst, nr, _) in items:
        for l in range(L):
            for r in range(nr):
                s = dst + r
                if l < int(active[s]):
                    assert torch.all(kv_k[l, s] == 0)
                    continue
                assert torch.equal(kv_k[l, s], pool[l, blk, 0, r])
                assert torch.equal(kv_v[l, s], pool[l, blk, 1, r])
                x = pool[l, blk, 0, r].double().numpy(force=True).reshape(1, kvw)
                want = O.rope(x, [int(slot_pos[s])], 500000.0, dh)[0]
                np.testing.assert_allclose(k_rot[l, s].double().numpy(force=True), want, atol=2e-2, rtol=1e-2)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_gather_rope_bulk_matches_register_path(N, dtype):
    """The TMA-staged K1 (bulk copies through shared memory, column chunks)
    writes exactly the bytes of the register-path kernel, including partial
    blocks and slots skipped at some layers."""
    L, kvw, dh = 4, 512, 128
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    code = N.BF16 if dtype == "bf16" else N.F32
    g = torch.Generator(device="cuda").manual_seed(5)
    pool = torch.randn((L, 9, 2, 16, kvw), device="cuda", generator=g).to(tdt)
    items = np.array([(3, 0, 16, 0), (7, 16, 16, 0), (1, 32, 10, 0), (5, 42, 1, 0), (0, 43, 16, 0)], dtype=np.int32)
    n = 59
    slot_pos = torch.randperm(200, device="cuda", generator=g)[:n].to(torch.int32)
    active = torch.zeros(n, dtype=torch.int32, device="cuda")
    active[[2, 17, 18, 42, 50]] = torch.tensor([1, 4, 2, 3, 1], dtype=torch.int32, device="cuda")
    half = dh // 2
    inv = torch.from_numpy(500000.0 ** (-2.0 * np.arange(half) / dh)).cuda()
    tab = torch.empty((256, half, 2), dtype=torch.float32, device="cuda")
    N.call("cc_rope_table", N.ptr(tab), N.ptr(inv), 256, half, code, N.stream_ptr())
    it = torch.from_numpy(items.reshape(-1)).cuda()
    outs = {}
    for mode in ((1, 0), (0, 0), (0, 128), (0, 256), (2, 0), (2, 128)):
        N.lib().cc_debug_k1(*mode)
        bufs = [torch.full((L, n, kvw), 7.0, dtype=tdt, device="cuda") for _ in range(3)]
        N.call("cc_gather_rope_kv", N.ptr(pool), pool.stride(0), pool.stride(1), N.ptr(it), len(items), 0, L,
               N.ptr(slot_pos), N.ptr(active), N.ptr(tab), *(N.ptr(b) for b in bufs), n * kvw, kvw, dh,
               code, N.stream_ptr())
        torch.cuda.synchronize()
        outs[mode] = bufs
    N.lib().cc_debug_k1(-1, -1)
    for mode, bufs in outs.items():
        for a, b in zip(bufs, outs[(1, 0)]):
            assert torch.equal(a, b), mode


def test_logits_argmax_first_max_wins(N):
    d, vocab = 64, 1000
    U = torch.zeros((vocab, d), dtype=torch.float32, device="cuda")
    U[17, 0] = 1.0
    U[900, 0] = 1.0  # tie -> first index
    h = torch.ones((1, d), dtype=torch.float32, device="cuda")
    logits = torch.empty((1, vocab), dtype=torch.float32, device="cuda")
    tok = torch.empty((1,), dtype=torch.int32, device="cuda")
    N.call("cc_logits_argmax", N.ptr(h), None, 1e-6, N.ptr(U), N.ptr(logits), N.ptr(tok), 1, d, vocab, N.F32,
           N.stream_ptr())
    assert int(tok.item()) == 17


@pytest.mark.parametrize("Hq,Hkv,dh", [(32, 8, 128), (4, 4, 64)])
def test_segment_mass_tensor_core_matches_simt(N, Hq, Hkv, dh):
    """K8a: the tcgen05 segment-mass kernel against the SIMT reference (fp64
    sums of the same softmax) and against torch fp32 probabilities."""
    n, nq = 900, 300
    g = torch.Generator(device="cuda").manual_seed(Hq)
    q_slot = torch.sort(torch.randperm(n, generator=g, device="cuda")[:nq]).values.int().contiguous()
    q = torch.randn((nq, Hq, dh), generator=g, device="cuda").bfloat16()
    k = torch.randn((n, Hkv, dh), generator=g, device="cuda").bfloat16()
    v = torch.randn((n, Hkv, dh), generator=g, device="cuda").bfloat16()
    pad = torch.zeros(n, dtype=torch.uint8, device="cuda")
    pad[250:256] = 1
    keep = pad[q_slot.long()] == 0
    q_slot, q = q_slot[keep].contiguous(), q[keep].contiguous()
    nq = q_slot.numel()
    ctx = torch.empty((nq, Hq * dh), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((nq, Hq), dtype=torch.float32, device="cuda")
    N.call("cc_attention", N.ptr(q), N.ptr(k), N.ptr(v), N.ptr(q_slot), N.ptr(pad), N.ptr(ctx), N.ptr(lse), nq, n, Hq,
           Hkv, dh, N.BF16, 0, N.stream_ptr())
    bounds = [0, 100, 250, 400, 401, 700, 900]
    lo = torch.tensor(bounds[:-1], dtype=torch.int32, device="cuda")
    hi = torch.tensor(bounds[1:], dtype=torch.int32, device="cuda")
    rows = torch.arange(0, nq, 3, dtype=torch.int32, device="cuda")
    n_seg = len(bounds) - 1
    out = {}
    for name, dt in (("tc", N.BF16), ("simt", N.F32)):
        mass = torch.zeros((rows.numel(), n_seg + 1), dtype=torch.float64, device="cuda")
        qq, kk = (q, k) if dt == N.BF16 else (q.float(), k.float())
        ll = lse if dt == N.BF16 else lse.float()
        N.call("cc_segment_mass", N.ptr(qq), N.ptr(kk), N.ptr(q_slot), N.ptr(pad), N.ptr(ll), N.ptr(lo), N.ptr(hi),
               n_seg, N.ptr(rows), rows.numel(), N.ptr(mass), n, Hq, Hkv, dh, dt, N.stream_ptr())
        torch.cuda.synchronize()
        out[name] = mass
    torch.testing.assert_close(out["tc"], out["simt"], atol=2e-3, rtol=2e-3)
    # rows of the softmax sum to one: segments cover every visible key
    torch.testing.assert_close(out["tc"][:, :n_seg].sum(dim=1), torch.ones(rows.numel(), dtype=torch.float64,
                                                                          device="cuda"), atol=3e-3, rtol=0)
    again = torch.zeros_like(out["tc"])
    N.call("cc_segment_mass", N.ptr(q), N.ptr(k), N.ptr(q_slot), N.ptr(pad), N.ptr(lse), N.ptr(lo), N.ptr(hi), n_seg,
           N.ptr(rows), rows.numel(), N.ptr(again), n, Hq, Hkv, dh, N.BF16, N.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(again, out["tc"])  # deterministic


def test_bf16_product_path_fails_loudly_on_unsupported_shapes(N):
    """No silent fallback: in bf16 the product path (impl 0) runs the tcgen05
    kernels (or the M <= 4 GEMV) only; a shape they do not support is an
    error, and no SIMT kernel ever runs on bf16 data unless asked (impl 2)."""
    from paper_2502_15734_b200.errors import NativeError

    before = N.bf16_simt_launches()
    A = torch.randn((64, 128), device="cuda").bfloat16()
    B = torch.randn((100, 128), device="cuda").bfloat16()  # N % 128 != 0
    C = torch.zeros((64, 100), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(NativeError, match="gemm_tc"):
        N.call("cc_gemm", N.ptr(A), 128, N.ptr(B), 128, N.ptr(C), 100, 64, 100, 128, N.EPI_STORE, N.BF16, 0,
               N.stream_ptr())
    q = torch.randn((8, 4, 32), device="cuda").bfloat16()  # d_head 32: no tcgen05 attention
    kv = torch.randn((64, 4, 32), device="cuda").bfloat16()
    rows = torch.arange(8, dtype=torch.int32, device="cuda")
    ctx = torch.empty((8, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((8, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(NativeError, match="attention_tc"):
        N.call("cc_attention", N.ptr(q), N.ptr(kv), N.ptr(kv), N.ptr(rows), None, N.ptr(ctx), N.ptr(lse), 8, 64, 4, 4,
               32, N.BF16, 0, N.stream_ptr())
    N.assert_tensor_core_only(before)
    # the explicit SIMT reference is counted
    N.call("cc_attention", N.ptr(q), N.ptr(kv), N.ptr(kv), N.ptr(rows), None, N.ptr(ctx), N.ptr(lse), 8, 64, 4, 4,
           32, N.BF16, 2, N.stream_ptr())
    torch.cuda.synchronize()
    assert N.bf16_simt_launches() == before + 1


@pytest.mark.parametrize("n", [8193, 20000, 131072])
def test_topk_select_long_chunks_radix_path(N, n):
    """Chunks longer than the shared-memory sort (8192) go through the radix
    select: same result as the reference's lexsort order, with heavy ties,
    signed zeros and negative scores."""
    import paper_2502_15734_b200 as cc
    from paper_2502_15734_b200.planner import recompute_count, select_tokens_batched

    r = np.random.default_rng(n)
    s = np.round(r.standard_normal(n), 2)
    s[r.choice(n, n // 10, replace=False)] = -0.0
    s[r.choice(n, n // 10, replace=False)] = 0.0
    for cfo in (1e-4, 0.15, 0.5, 1.0):
        k = recompute_count(n, cfo)
        want = np.sort(np.lexsort((np.arange(n), -s))[:k])
        np.testing.assert_array_equal(cc.select_tokens(s, cfo), want)
    # batched with a short chunk (both kernels' inputs in one launch)
    short = np.round(r.standard_normal(300), 1)
    got = select_tokens_batched([short, s], [recompute_count(300, 0.2), recompute_count(n, 0.2)])
    np.testing.assert_array_equal(got[0], np.sort(np.lexsort((np.arange(300), -short))[:60]))
    np.testing.assert_array_equal(got[1], np.sort(np.lexsort((np.arange(n), -s))[:recompute_count(n, 0.2)]))


@pytest.mark.parametrize("M,Hq,Hkv,d,n_slots", [(802, 32, 8, 4096, 5152), (400, 32, 8, 4096, 5152), (150, 8, 2, 512, 700),
                                                 (300, 8, 1, 1024, 900), (40, 8, 2, 512, 300)])
def test_gemm_qkv_rope_fused_matches_unfused(N, M, Hq, Hkv, d, n_slots):
    """K3: the QKV GEMM with RoPE + K/V scatter in its CTA-pair epilogue
    (cc_gemm_qkv_rope) gives the same bits as the GEMM followed by
    cc_rope_scatter_qkv, and matches a torch fp32 reference within bf16.
    M = 40 and 802 are outside the fused kernel's range (64..512 rows): the
    GEMM + rope_scatter composition runs there."""
    dh = 128
    g = torch.Generator(device="cuda").manual_seed(M + Hq)
    NQ = (Hq + 2 * Hkv) * dh
    x = (torch.randn((M, d), generator=g, device="cuda") * 0.5).bfloat16()
    w = (torch.randn((NQ, d), generator=g, device="cuda") / d ** 0.5).bfloat16()
    slots = torch.sort(torch.randperm(n_slots, generator=g, device="cuda")[:M]).values.int().contiguous()
    pos = (slots + 7).int().contiguous()
    inv = 1.0 / (500000.0 ** (torch.arange(0, dh // 2, dtype=torch.float64) * 2 / dh))
    ang = torch.arange(n_slots + 8, dtype=torch.float64)[:, None] * inv[None, :]
    table = torch.stack([torch.cos(ang), torch.sin(ang)], dim=-1).float().cuda().contiguous()
    kvw = Hkv * dh

    def bufs():
        return (torch.zeros((M, Hq * dh), dtype=torch.bfloat16, device="cuda"),
                *[torch.zeros((n_slots, kvw), dtype=torch.bfloat16, device="cuda") for _ in range(3)])

    fq, fk, fv, fkr = bufs()
    qkv = torch.empty((M, NQ), dtype=torch.bfloat16, device="cuda")
    N.call("cc_gemm_qkv_rope", N.ptr(x), d, N.ptr(w), d, M, d, N.ptr(slots), N.ptr(pos), N.ptr(table), N.ptr(fq),
           N.ptr(fk), N.ptr(fv), N.ptr(fkr), N.ptr(qkv), Hq, Hkv, dh, N.BF16, N.stream_ptr())
    uq, uk, uv, ukr = bufs()
    # (impl 4: no K split, as the fused kernel; below its range the composition runs impl 0)
    N.call("cc_gemm", N.ptr(x), d, N.ptr(w), d, N.ptr(qkv), NQ, M, NQ, d, N.EPI_STORE, N.BF16, 4 if M >= 64 else 0,
           N.stream_ptr())
    N.call("cc_rope_scatter_qkv", N.ptr(qkv), NQ, M, N.ptr(slots), N.ptr(pos), N.ptr(table), N.ptr(uq), N.ptr(uk),
           N.ptr(uv), N.ptr(ukr), Hq, Hkv, dh, N.BF16, N.stream_ptr())
    torch.cuda.synchronize()
    for a, b in ((fq, uq), (fk, uk), (fv, uv), (fkr, ukr)):
        assert torch.equal(a, b)
    # torch fp32 reference (rotate-half RoPE at pos)
    ref = x.float() @ w.float().T
    cs = table[pos.long()]  # [M][64][2]

    def rot(t):  # t [M][h][128]
        a, b = t[..., :64], t[..., 64:]
        c, s = cs[:, None, :, 0], cs[:, None, :, 1]
        return torch.cat([a * c - b * s, a * s + b * c], dim=-1)

    q = rot(ref[:, : Hq * dh].view(M, Hq, dh)).reshape(M, -1)
    k = ref[:, Hq * dh: Hq * dh + kvw]
    kr = rot(k.view(M, Hkv, dh)).reshape(M, -1)
    v = ref[:, Hq * dh + kvw:]
    sl = slots.long()
    for got, want in ((fq, q), (fk[sl], k), (fkr[sl], kr), (fv[sl], v)):
        torch.testing.assert_close(got.float(), want, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("Hq,Hkv,dh,n,n_rows", [(32, 8, 128, 3001, 1200), (16, 2, 64, 2013, 900), (8, 1, 128, 4099, 2000)])
def test_attention_many_rows_and_ragged_keys(N, Hq, Hkv, dh, n, n_rows):
    """The default (ping-pong) attention kernel on grids of more than one
    wave (no key splits), key counts that are not a multiple of 16 and pads in
    several places, against torch fp32; and run-to-run bit-identical."""
    g = torch.Generator(device="cuda").manual_seed(n + dh)
    rows = torch.sort(torch.randperm(n, generator=g, device="cuda")[:n_rows]).values.int()
    q = torch.randn((n_rows, Hq, dh), generator=g, device="cuda").bfloat16()
    k = torch.randn((n, Hkv, dh), generator=g, device="cuda").bfloat16()
    v = torch.randn((n, Hkv, dh), generator=g, device="cuda").bfloat16()
    pad = torch.zeros(n, dtype=torch.uint8, device="cuda")
    pad[7:9] = 1
    pad[1000:1013] = 1
    pad[n - 5: n - 1] = 1
    rows = rows[pad[rows.long()] == 0].contiguous()
    q = q[: rows.numel()].contiguous()
    outs = []
    for _ in range(2):
        ctx = torch.empty((rows.numel(), Hq * dh), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((rows.numel(), Hq), dtype=torch.float32, device="cuda")
        N.call("cc_attention", N.ptr(q), N.ptr(k), N.ptr(v), N.ptr(rows), N.ptr(pad), N.ptr(ctx), N.ptr(lse),
               rows.numel(), n, Hq, Hkv, dh, N.BF16, 0, N.stream_ptr())
        torch.cuda.synchronize()
        outs.append((ctx, lse))
    ref, ref_lse = _attn_ref(q, k, v, rows, pad, Hq, Hkv)
    torch.testing.assert_close(outs[0][0].float(), ref, atol=3e-2, rtol=3e-2)
    torch.testing.assert_close(outs[0][1], ref_lse, atol=2e-3, rtol=1e-3)
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
