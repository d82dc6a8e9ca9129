"""A/B of the tcgen05 attention kernel shapes (cc_debug_attn_variant) on the
BASELINE configs' attention problems, timed with CUDA events on the launching
stream (median of `iters` launches after warm-up), each variant checked
against variant 0 and a torch fp32 reference.

  python tools/attn_ab.py [variants=0,1,2] [iters=50]
"""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_15734_b200 import _native as N  # noqa: E402

# variant specs: "v" or "v@target/parts" (forced key split, CCB_ATTN_SPLIT)
lib = N.lib()
lib.cc_debug_attn_variant.argtypes = [ctypes.c_int]

CASES = {  # name: (n_q recomputed rows, n_keys, Hq, Hkv)
    "config2 r=.15": (802, 5152, 32, 8),
    "config2 r=.05": (290, 5152, 32, 8),
    "config2 full": (5152, 5152, 32, 8),
    "config5 32k": (4960, 32800, 32, 8),
    "config4 70B rank": (2496, 16416, 8, 1),
}


def make(n_q, n, Hq, Hkv, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if n_q == n:
        rows = torch.arange(n, dtype=torch.int32, device="cuda")
    else:  # question rows at the end + the rest spread uniformly (config-2 layout)
        rest = torch.sort(torch.randperm(n - 32, generator=g, device="cuda")[: n_q - 32]).values
        rows = torch.cat([rest, torch.arange(n - 32, n, device="cuda")]).int()
    q = torch.randn((n_q, Hq, 128), generator=g, device="cuda").bfloat16()
    k = torch.randn((n, Hkv, 128), generator=g, device="cuda").bfloat16()
    v = torch.randn((n, Hkv, 128), generator=g, device="cuda").bfloat16()
    return rows.contiguous(), q, k, v


def run(args, ctx, lse):
    rows, q, k, v = args
    n_q, Hq = q.shape[0], q.shape[1]
    n, Hkv = k.shape[0], k.shape[1]
    N.call("cc_attention", N.ptr(q), N.ptr(k), N.ptr(v), N.ptr(rows), None, N.ptr(ctx), N.ptr(lse), n_q, n, Hq, Hkv,
           128, N.BF16, 1, N.stream_ptr())


def ref(args):
    rows, q, k, v = args
    Hq, Hkv = q.shape[1], k.shape[1]
    G = Hq // Hkv
    kk = k.float().repeat_interleave(G, dim=1)
    vv = v.float().repeat_interleave(G, dim=1)
    out = []
    for i0 in range(0, q.shape[0], 256):
        qq = q[i0:i0 + 256].float()
        s = torch.einsum("qhd,khd->hqk", qq, kk) / 128 ** 0.5
        mask = torch.arange(k.shape[0], device="cuda")[None, :] > rows[i0:i0 + 256, None].long()
        s.masked_fill_(mask[None], float("-inf"))
        out.append(torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), vv).reshape(qq.shape[0], -1))
    return torch.cat(out)


def main():
    variants = (sys.argv[1] if len(sys.argv) > 1 else "0,1,2").split(",")
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    cases_sel = sys.argv[3].split(",") if len(sys.argv) > 3 else None
    for name, (n_q, n, Hq, Hkv) in CASES.items():
        if cases_sel and not any(c in name for c in cases_sel):
            continue
        args = make(n_q, n, Hq, Hkv)
        keys_vis = (args[0].long() + 1).sum().item()
        flop = 4.0 * Hq * 128 * keys_vis
        ctx0 = None
        want = ref(args) if n_q * n * Hq <= 6e9 else None
        line = [f"{name:18s} flop {flop / 1e9:7.1f}G"]
        for spec in variants:
            # spec: "v", "vxE" (timing experiment E, CCB_ATTN_EXP), "...@target/parts" (CCB_ATTN_SPLIT)
            os.environ.pop("CCB_ATTN_EXP", None)
            os.environ.pop("CCB_ATTN_SPLIT", None)
            head = spec.split("@")[0]
            if "x" in head:
                os.environ["CCB_ATTN_EXP"] = head.split("x")[1]
            if "@" in spec:
                os.environ["CCB_ATTN_SPLIT"] = spec.split("@")[1].replace("/", ",")
            lib.cc_debug_attn_variant(int(head.split("x")[0]))
            ctx = torch.empty((n_q, Hq * 128), dtype=torch.bfloat16, device="cuda")
            lse = torch.empty((n_q, Hq), dtype=torch.float32, device="cuda")
            for _ in range(3):
                run(args, ctx, lse)
            torch.cuda.synchronize()
            ev = []
            for _ in range(iters):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                run(args, ctx, lse)
                b.record()
                ev.append((a, b))
            torch.cuda.synchronize()
            us = statistics.median(x.elapsed_time(y) for x, y in ev) * 1e3
            err = ""
            if want is not None:
                err = f" err {((ctx.float() - want).norm() / want.norm()).item():.1e}"
            if ctx0 is None:
                ctx0 = ctx.clone()
            line.append(f"v{spec} {us:7.1f}us {flop / us / 1e6:6.0f}TF/s{err}")
        lib.cc_debug_attn_variant(-1)
        os.environ.pop("CCB_ATTN_EXP", None)
        os.environ.pop("CCB_ATTN_SPLIT", None)
        print(" | ".join(line), flush=True)


if __name__ == "__main__":
    main()
