"""Device execution of the chunk-cache fix-up prefill (model.py:348-442).

Data layout in HBM for one request (n slots, L layers, kvw = Hkv * dh):
  * ``hidden`` [n_rows, d] f32 (f64 in fp64 mode): residual stream of the
    rows whose Q/K/V are ever recomputed, ordered by (-depth, slot) so the
    rows active at layer l are always the prefix ``hidden[:n_act[l]]``.
  * ``kv_k`` / ``kv_v`` [L, n, kvw]: the returned position-free KV (cached
    rows copied from the pool, active rows freshly computed = cache repair).
  * ``k_rot`` [L, n, kvw]: keys rotated at their slot position for attention.
Per layer: RMSNorm -> QKV GEMM -> RoPE/scatter -> attention -> o_proj GEMM
(+residual) -> RMSNorm -> gate/up GEMM (+SwiGLU or GELU) -> down GEMM
(+residual).  One K1 launch gathers+rotates every cached block for all
layers before the loop.  Every tensor op is a CUDA kernel from
libcc_b200.so; torch only allocates memory and provides the stream.
"""

from __future__ import annotations

import contextlib
import os

import numpy as np

from . import _native as N
from .errors import PlanError, ShapeError
from .model import BLOCK, FULL_DEPTH, AttentionRecord, ChunkCache, KVCache, Model, PrefillResult, _Payload

_GATHER_DT = np.dtype([("src_block", "<i4"), ("dst_slot", "<i4"), ("n_rows", "<i4"), ("pad", "<i4")])


class DevicePlan:
    """Host-resolved index arrays of one request, uploaded in a single copy."""

    def __init__(self, model: Model, token_ids, positions, is_pad, mask, depth, seg_slots, seg_caches, question_span):
        import torch

        cfg = model.config
        L = cfg.n_layers
        n = int(token_ids.size)
        self.n = n
        depth_eff = np.where(depth == FULL_DEPTH, L, depth).astype(np.int64)
        rows = np.flatnonzero(mask)
        order = np.argsort(-depth_eff[rows], kind="stable")
        rows = rows[order]
        self.rows = rows  # slot of each hidden row, (-depth, slot) order
        self.n_rows = int(rows.size)
        rd = depth_eff[rows]
        self.row_depth = rd.copy()
        self.n_act = [int(np.count_nonzero(rd > l)) for l in range(L)]
        self.row_pos = positions[rows].astype(np.int32)
        self.row_tok = token_ids[rows].astype(np.int32)
        self.active_until_h = np.where(mask, depth_eff, 0).astype(np.int32)
        active_until = np.where(mask, depth_eff, 0).astype(np.int32)
        key_pos = np.where(is_pad, 0, positions).astype(np.int32)
        self.max_pos = int(key_pos.max()) + 1 if n else 1
        items, host_items = [], []
        self.host_payloads = []  # host-tier payloads, in staging-slot order
        n_host_blocks = 0
        for (start, _), payload in zip(seg_slots, seg_caches):
            if payload is None:
                continue
            is_host = getattr(payload, "tier", "hbm") == "host"
            nb = payload.n_blocks if is_host else len(payload.blocks)
            for b in range(nb):
                nr = min(BLOCK, payload.n_slots - BLOCK * b)
                if nr <= 0:
                    continue
                if is_host:  # block b of this payload sits at staging block n_host_blocks + b
                    host_items.append((n_host_blocks + b, start + BLOCK * b, nr, 0))
                else:
                    items.append((int(payload.blocks[b]), start + BLOCK * b, nr, 0))
            if is_host:
                self.host_payloads.append((payload, n_host_blocks))
                n_host_blocks += payload.n_blocks
        self.items = np.array(items, dtype=_GATHER_DT)
        self.n_items = len(items)
        self.host_items = np.array(host_items, dtype=_GATHER_DT)
        self.n_host_items = len(host_items)
        self.n_host_blocks = n_host_blocks
        self.n_cached_rows = int(sum(it[2] for it in items)) + int(sum(it[2] for it in host_items))
        cached = np.zeros(n, bool)
        for (src, dst, nr, _) in list(items) + list(host_items):
            cached[dst:dst + nr] = True
        self.cached_active = [int(np.count_nonzero(cached & (active_until > l))) for l in range(L)]
        # keys visible per active row (slot <= own slot, not pad) -> attention FLOPs
        nonpad_before = np.cumsum(~np.asarray(is_pad, bool))
        vis = nonpad_before[rows] if rows.size else np.zeros(0, np.int64)
        self.attn_keys = [int(vis[: self.n_act[l]].sum()) for l in range(L)]
        # pack every int32 array into one host buffer -> one H2D copy
        parts = {
            "row_slot": rows.astype(np.int32),
            "row_pos": positions[rows].astype(np.int32),
            "row_tok": token_ids[rows].astype(np.int32),
            "slot_pos": key_pos,
            "active_until": active_until,
            "items": self.items.view(np.int32).reshape(-1),
            "host_items": self.host_items.view(np.int32).reshape(-1),
        }
        self.stats_segments = None
        self.stats_rows = np.zeros(0, np.int32)
        self.stats_keys = 0.0
        offs, cur = {}, 0
        for k, a in parts.items():
            offs[k] = (cur, a.size)
            cur += -(-max(a.size, 1) // 4) * 4  # keep 16-byte alignment
        host = np.zeros(cur, np.int32)
        for k, a in parts.items():
            o, s = offs[k]
            host[o:o + s] = a
        pad_bytes = -(-n // 16) * 16
        host_pad = np.zeros(pad_bytes, np.uint8)
        host_pad[:n] = is_pad
        self.h2d_bytes = host.nbytes + host_pad.nbytes
        pin = torch.from_numpy(host).pin_memory()
        dev = pin.to(model.device, non_blocking=True)
        pin_pad = torch.from_numpy(host_pad).pin_memory()
        self.key_pad = pin_pad.to(model.device, non_blocking=True)
        self.has_pad = bool(is_pad.any())
        self._keep = (pin, pin_pad)
        self.d = {k: dev[o:o + s] for k, (o, s) in offs.items()}


class LazyAttention:
    """Device operands kept per layer to materialise softmax weights."""

    def __init__(self, model, plan, k_rot):
        self.model, self.plan, self.k_rot = model, plan, k_rot
        self.q = {}
        self.lse = {}
        # row order of each recorded layer (an online focus cut permutes the
        # hidden rows mid-prefill: earlier layers keep the order they ran in)
        self.rows = {}
        self.row_slot = {}

    def materialize(self, layer: int) -> np.ndarray:
        import torch

        cfg = self.model.kcfg
        H = cfg.n_heads
        rows = self.rows.get(layer, self.plan.rows[: self.plan.n_act[layer]])
        n_l = rows.size
        if n_l == 0:
            return np.zeros((H, 0, self.plan.n))
        slot = self.row_slot.get(layer, self.plan.d["row_slot"])
        probs = torch.empty((H, n_l, self.plan.n), dtype=self.model.hidden_dtype, device=self.model.device)
        N.call("cc_attention_probs", N.ptr(self.q[layer]), N.ptr(self.k_rot[layer]), N.ptr(slot),
               N.ptr(self.plan.key_pad) if self.plan.has_pad else None, N.ptr(self.lse[layer]), N.ptr(probs), n_l,
               self.plan.n, H, cfg.kv_heads(), cfg.head_dim(), self.model.dtype_code, N.stream_ptr())
        order = np.argsort(rows, kind="stable")
        return probs.double().cpu().numpy()[:, order]

    def materialize_all(self) -> list:
        if not self.q:
            raise PlanError("attention weights were not recorded; call prefill(..., record_attention=True)")
        return [self.materialize(l) for l in range(self.model.config.n_layers)]


def _workspace(model: Model, plan: DevicePlan):
    import torch

    cfg = model.kcfg
    L, n, nr = cfg.n_layers, plan.n, max(plan.n_rows, 1)
    T, Hd = model.torch_dtype, model.hidden_dtype
    d, q, kv, ff = cfg.d_model, cfg.q_width(), cfg.kv_width(), cfg.ff_dim()
    dev = model.device
    e = torch.empty
    tp = model.tp is not None and model.tp.world > 1
    return {
        "partial": e((nr, d), dtype=Hd, device=dev) if tp else None,
        "hidden": e((nr, d), dtype=Hd, device=dev),
        "kv_k": e((L, n, kv), dtype=T, device=dev),
        "kv_v": e((L, n, kv), dtype=T, device=dev),
        "k_rot": e((L, n, kv), dtype=T, device=dev),
        "xn": e((nr, d), dtype=T, device=dev),
        "qkv": e((nr, q + 2 * kv), dtype=T, device=dev),
        "q_rot": e((nr, q), dtype=T, device=dev),
        "ctx": e((nr, q), dtype=T, device=dev),
        "act": e((nr, ff), dtype=T, device=dev),
        "lse": e((nr, cfg.n_heads), dtype=Hd, device=dev),
    }


class _HostPreload:
    """Layer-wise preloading of host-tier chunk caches (tiers.py, PAPER.md
    Algorithm 2): the copy engine fills a ring of ``L_p + 1`` HBM layer slots
    on a side stream (one DMA per host payload per layer); layer l's K1
    gather waits for its slot's copy event and its completion frees the slot
    for layer l + L_p + 1.  Copies of later layers overlap the compute of
    earlier ones; nothing on the SMs waits on PCIe."""

    def __init__(self, model: Model, plan: DevicePlan):
        import torch

        from .tiers import preload_depth

        cfg = model.kcfg
        self.L = cfg.n_layers
        self.plan = plan
        layer_bytes = sum(p.nbytes() for p, _ in plan.host_payloads) / self.L
        t_load = layer_bytes / model.h2d_bytes_per_s
        t_prefill = _estimate_layer_seconds(model, plan)
        self.depth = preload_depth(self.L, t_prefill, t_load)
        self.slots = min(self.L, self.depth + 1)
        self.staging = torch.empty((self.slots, plan.n_host_blocks, 2, BLOCK, cfg.kv_width()),
                                   dtype=model.torch_dtype, device=model.device)
        self.stream = model.copy_stream()
        self.staging.record_stream(self.stream)
        self.copied = [torch.cuda.Event() for _ in range(self.L)]
        self.free = [torch.cuda.Event() for _ in range(self.L)]
        start = torch.cuda.Event()
        start.record()  # buffers allocated / last used on the main stream
        self.stream.wait_event(start)
        self.bytes = 0
        for l in range(self.slots):
            self._copy(l)

    def _copy(self, l: int):
        import torch

        if l >= self.L:
            return
        slot = self.staging[l % self.slots]
        with torch.cuda.stream(self.stream):
            if l >= self.slots:
                self.stream.wait_event(self.free[l - self.slots])
            for p, off in self.plan.host_payloads:
                slot[off:off + p.n_blocks].copy_(p.data[l], non_blocking=True)
                self.bytes += p.nbytes() // self.L
            self.copied[l].record(self.stream)

    def gather(self, model: Model, plan: DevicePlan, ws: dict, l: int, rope, s):
        import torch

        cfg = model.kcfg
        torch.cuda.current_stream().wait_event(self.copied[l])
        st = self.staging[l % self.slots]
        N.call("cc_gather_rope_kv", N.ptr(st), 0, st.stride(0), N.ptr(plan.d["host_items"]), plan.n_host_items, l,
               l + 1, N.ptr(plan.d["slot_pos"]), N.ptr(plan.d["active_until"]), N.ptr(rope), N.ptr(ws["kv_k"]),
               N.ptr(ws["kv_v"]), N.ptr(ws["k_rot"]), plan.n * cfg.kv_width(), cfg.kv_width(), cfg.head_dim(),
               model.dtype_code, s)
        self.free[l].record()
        self._copy(l + self.slots)


class _L2Prefetch:
    """Side-stream L2 prefetch of a projection's weights (cc_prefetch_l2): the
    o_proj GEMM otherwise starts on cold weights (measured 38 us in the step
    vs 30 us L2-warm at config 2).  Weights are read-only, so the side stream
    needs no ordering against the main stream."""

    def __init__(self, model: Model):
        self.stream = model.copy_stream()

    def prefetch(self, w):
        N.call("cc_prefetch_l2", N.ptr(w), w.numel() * w.element_size(), self.stream.cuda_stream)


def _estimate_layer_seconds(model: Model, plan: DevicePlan) -> float:
    """Per-layer compute estimate of a plan for the preload depth: linear
    FLOPs at ~1 PFLOP/s plus attention FLOPs at ~0.45 PFLOP/s (the rates
    measured for these kernels on B200)."""
    cfg = model.kcfg
    d, q, kv, ff = cfg.d_model, cfg.q_width(), cfg.kv_width(), cfg.ff_dim()
    m = 3 if cfg.mlp == "swiglu" else 2
    rows = sum(plan.n_act) / max(1, cfg.n_layers)
    lin = 2.0 * rows * (d * (q + 2 * kv) + q * d + m * d * ff)
    att = 4.0 * cfg.n_heads * cfg.head_dim() * sum(plan.attn_keys) / max(1, cfg.n_layers)
    return max(lin / 1.0e15 + att / 0.45e15, 1e-6)


def _record_default(model: Model, plan: DevicePlan) -> bool:
    cfg = model.kcfg
    bytes_q = sum(plan.n_act) * cfg.q_width() * model.torch_dtype.itemsize
    return plan.n <= 8192 and bytes_q <= (256 << 20)


class KernelTimer:
    """CUDA events around each launch family on the launching stream (bench
    instrumentation: per-kernel average durations inside the timed region)."""

    def __init__(self):
        self.events = {}
        self.flops = {}
        self.bytes = {}

    def span(self, name, flops=0.0, nbytes=0.0):
        import torch

        t = self

        class _Span:
            def __enter__(self_inner):
                self_inner.a = torch.cuda.Event(enable_timing=True)
                self_inner.a.record()

            def __exit__(self_inner, *exc):
                b = torch.cuda.Event(enable_timing=True)
                b.record()
                t.events.setdefault(name, []).append((self_inner.a, b))
                t.flops[name] = t.flops.get(name, 0.0) + flops
                t.bytes[name] = t.bytes.get(name, 0.0) + nbytes

        return _Span()

    def summary(self):
        out = {}
        for k, ev in self.events.items():
            ms = sum(a.elapsed_time(b) for a, b in ev)
            out[k] = {"launches": len(ev), "ms_total": ms, "flops": self.flops[k], "bytes": self.bytes[k]}
        return out


class _NoTimer:
    class _Null:
        def __enter__(self):
            return None

        def __exit__(self, *exc):
            return False

    _n = _Null()

    def span(self, name, flops=0.0, nbytes=0.0):
        return self._n


_NOTIMER = _NoTimer()


class OnlineFocus:
    """Single-pass focused-chunk early termination (reference:
    harness.py:406-428 runs prefill twice).  After each layer the question
    rows' head-mean mass per chunk (K8a) feeds Algorithm 1 (planner.
    FocusTracker); when it fires with cutoff L* < L, the recompute rows of the
    unfocused cached chunks stop at layer L* — the same depths the reference's
    second pass uses, so the layers it recomputes are identical."""

    def __init__(self, request, window: int, n_layers: int):
        from .planner import FocusTracker

        self.k = len(request.segments)
        self.tracker = FocusTracker(self.k, window, n_layers)
        self.n_layers = n_layers
        self.request = request
        self.result = None
        self.cut = False
        self.q_span = tuple(request.question_span)

    def cut_slots(self, focused) -> np.ndarray:
        out = []
        for i, (seg, (s0, _)) in enumerate(zip(self.request.segments, self.request.segment_slots)):
            if seg.cache is None or i in focused or seg.recompute is None:
                continue
            idx = np.flatnonzero(np.asarray(seg.recompute, dtype=bool))
            if idx.size:
                out.append(s0 + idx)
        return np.concatenate(out) if out else np.zeros(0, np.int64)


def _apply_cut(model, plan, ws, slots, new_depth):
    """Deactivate hidden rows of ``slots`` from layer ``new_depth`` on: permute
    rows so the active ones stay a prefix, refresh the device index arrays and
    re-gather the stale cached K/V of those slots for the remaining layers."""
    import torch

    L = model.config.n_layers
    is_cut = np.isin(plan.rows, slots)
    plan.row_depth = np.where(is_cut, np.minimum(plan.row_depth, new_depth), plan.row_depth)
    perm = np.argsort(-plan.row_depth, kind="stable")
    plan.rows, plan.row_depth = plan.rows[perm], plan.row_depth[perm]
    plan.row_pos, plan.row_tok = plan.row_pos[perm], plan.row_tok[perm]
    plan.n_act = [int(np.count_nonzero(plan.row_depth > l)) for l in range(L)]
    dev = model.device
    h = ws["hidden"]
    idx = torch.from_numpy(perm.astype(np.int64)).to(dev)
    h[: plan.n_rows].copy_(h[: plan.n_rows].index_select(0, idx))
    plan.d["row_slot"].copy_(torch.from_numpy(plan.rows.astype(np.int32)).to(dev))
    plan.d["row_pos"].copy_(torch.from_numpy(plan.row_pos).to(dev))
    plan.active_until_h[slots] = np.minimum(plan.active_until_h[slots], new_depth)
    plan.d["active_until"].copy_(torch.from_numpy(plan.active_until_h).to(dev))
    if getattr(plan, "stats_row_spans", None):
        _attach_stats_rows(model, plan, plan.stats_row_spans)
        # stats rows of spans containing cut slots hold no valid mass from new_depth on
        cut_rows, off = [], 0
        for lo, hi in plan.stats_row_spans:
            if np.any((slots >= lo) & (slots < hi)):
                cut_rows.extend(range(off, off + hi - lo))
            off += hi - lo
        if cut_rows:
            import torch as _t

            prev = getattr(plan, "stats_cut_rows", [])
            plan.stats_cut_rows = prev + [(_t.tensor(cut_rows, device=dev), new_depth)]
    # stale rows of the cut slots for layers >= new_depth (K1 on the affected blocks only)
    touched = [it for it in plan.items if np.any((slots >= it["dst_slot"]) & (slots < it["dst_slot"] + it["n_rows"]))]
    if touched and new_depth < L:
        items = torch.from_numpy(np.array(touched, dtype=_GATHER_DT).view(np.int32).reshape(-1).copy()).to(dev)
        cfg = model.kcfg
        pool = model.pool
        N.call("cc_gather_rope_kv", N.ptr(pool.storage), pool.layer_stride, pool.block_stride, N.ptr(items),
               len(touched), new_depth, L, N.ptr(plan.d["slot_pos"]), N.ptr(plan.d["active_until"]),
               N.ptr(model.rope_table(plan.max_pos)), N.ptr(ws["kv_k"]), N.ptr(ws["kv_v"]), N.ptr(ws["k_rot"]),
               plan.n * cfg.kv_width(), cfg.kv_width(), cfg.head_dim(), model.dtype_code, N.stream_ptr())


@contextlib.contextmanager
def concurrent_streams():
    """Serving mode: requests may be in flight on several CUDA streams at
    once.  Every kernel here already keeps per-stream scratch; inside this
    context the GEMMs also run without stream-K tails, whose folds spin on
    sibling CTAs (two such GEMMs on different streams could each hold SMs
    waiting for CTAs no SM is free to run)."""
    prev = N.lib().cc_set_stream_k(0)
    try:
        yield
    finally:
        N.lib().cc_set_stream_k(prev)


def execute(model: Model, plan: DevicePlan, ws: dict, **kw):
    """Launch the per-layer pipeline (see _execute) with programmatic dependent
    launch enabled for its kernels when model.prefill_pdl."""
    prev = N.lib().cc_set_pdl(1 if getattr(model, "prefill_pdl", False) else 0)
    try:
        return _execute(model, plan, ws, **kw)
    finally:
        N.lib().cc_set_pdl(prev)


def _execute(model: Model, plan: DevicePlan, ws: dict, *, record=False, record_values=False, stats=False,
             gemm_impl=0, attn_impl=0, timer=None, focus: OnlineFocus | None = None):
    """Launch the per-layer pipeline on the current stream.  Returns the
    LazyAttention (if recording), value trace list and stats masses.
    Under tensor parallelism (model.tp) the o_proj and down_proj GEMMs write
    rank-partial outputs that are all-reduced before the residual add."""
    import torch

    cfg = model.kcfg
    tp = model.tp if (model.tp is not None and model.tp.world > 1) else None
    part = ws.get("partial")
    L, n = cfg.n_layers, plan.n
    H, Hkv, dh, d = cfg.n_heads, cfg.kv_heads(), cfg.head_dim(), cfg.d_model
    qw, kvw, ff = cfg.q_width(), cfg.kv_width(), cfg.ff_dim()
    dt = model.dtype_code
    s = N.stream_ptr()
    P = N.ptr
    D = plan.d
    pool = model.pool
    rope = model.rope_table(plan.max_pos)
    hidden, kv_k, kv_v, k_rot = ws["hidden"], ws["kv_k"], ws["kv_v"], ws["k_rot"]
    xn, qkv, q_rot, ctx, act, lse = ws["xn"], ws["qkv"], ws["q_rot"], ws["ctx"], ws["act"], ws["lse"]
    if plan.n_rows:
        N.call("cc_embed_rows", P(model.w["embed"]), P(D["row_tok"]), P(hidden), plan.n_rows, d, dt, s)
    tm = _NOTIMER if timer is None else timer
    esz = model.torch_dtype.itemsize
    if plan.n_items:
        # algorithmic bytes: read K,V block rows, write kv_k, kv_v, k_rot (rows not recomputed at that layer)
        moved = sum(plan.n_cached_rows - plan.cached_active[l] for l in range(L)) * kvw * esz * 5
        with tm.span("gather_rope", nbytes=moved):
            N.call("cc_gather_rope_kv", P(pool.storage), pool.layer_stride, pool.block_stride, P(D["items"]),
                   plan.n_items, 0, L, P(D["slot_pos"]), P(D["active_until"]), P(rope), P(kv_k), P(kv_v), P(k_rot),
                   n * kvw, kvw, dh, dt, s)
    preload = _HostPreload(model, plan) if plan.n_host_items else None
    l2pf = _L2Prefetch(model) if (dt == N.BF16 and model.l2_prefetch) else None
    lazy = LazyAttention(model, plan, k_rot) if record else None
    vtrace = [] if record_values else None
    n_stats = plan.stats_rows.size if stats else 0
    n_seg = len(plan.stats_segments) if (stats and plan.stats_segments) else 0
    mass = torch.zeros((L, max(n_stats, 1), n_seg + 1), dtype=torch.float64, device=model.device) if n_stats else None
    key_pad = P(plan.key_pad) if plan.has_pad else None
    eps = cfg.rms_eps
    for l in range(L):
        lw = model.w["layers"][l]
        n_l = plan.n_act[l]
        if n_l == 0:
            if preload is not None:  # nothing computed at this layer: the cached rows still land
                preload.gather(model, plan, ws, l, rope, s)
            if record_values:
                vtrace.append((kv_v[l], None, None))
            continue
        with tm.span("rmsnorm", nbytes=n_l * d * (4 + esz)):
            N.call("cc_rmsnorm", P(hidden), P(xn), P(lw.get("attn_norm")), n_l, d, eps, dt, s)
        if gemm_impl == 0:
            # QKV GEMM with RoPE and the K/V scatter in its epilogue (K3; bf16
            # shapes it covers, else the same GEMM + rope_scatter, bit-identical)
            with tm.span("gemm", flops=2.0 * n_l * (qw + 2 * kvw) * d):
                N.call("cc_gemm_qkv_rope", P(xn), d, P(lw["w_qkv"]), d, n_l, d, P(D["row_slot"]), P(D["row_pos"]),
                       P(rope), P(q_rot), P(kv_k[l]), P(kv_v[l]), P(k_rot[l]), P(qkv), H, Hkv, dh, dt, s)
        else:
            with tm.span("gemm", flops=2.0 * n_l * (qw + 2 * kvw) * d):
                N.call("cc_gemm", P(xn), d, P(lw["w_qkv"]), d, P(qkv), qw + 2 * kvw, n_l, qw + 2 * kvw, d,
                       N.EPI_STORE, dt, gemm_impl, s)
            # algorithmic bytes: read the qkv row, write q_rot and k, k_rot, v at the row slots
            with tm.span("rope_scatter", nbytes=n_l * (qw + 2 * kvw + qw + 3 * kvw) * esz):
                N.call("cc_rope_scatter_qkv", P(qkv), qw + 2 * kvw, n_l, P(D["row_slot"]), P(D["row_pos"]), P(rope),
                       P(q_rot), P(kv_k[l]), P(kv_v[l]), P(k_rot[l]), H, Hkv, dh, dt, s)
        if preload is not None:
            preload.gather(model, plan, ws, l, rope, s)
        if l2pf is not None:  # o_proj weights -> L2 while attention runs (it reads K/V from L2 only)
            l2pf.prefetch(lw["w_o"])
        with tm.span("attention", flops=4.0 * H * dh * plan.attn_keys[l]):
            N.call("cc_attention", P(q_rot), P(k_rot[l]), P(kv_v[l]), P(D["row_slot"]), key_pad, P(ctx), P(lse), n_l,
                   n, H, Hkv, dh, dt, attn_impl, s)
        if n_stats:
            # algorithmic FLOPs: q.k over every causal key of each stats row
            with tm.span("segment_mass", flops=2.0 * H * dh * plan.stats_keys):
                N.call("cc_segment_mass", P(q_rot), P(k_rot[l]), P(D["row_slot"]), key_pad, P(lse), P(D["seg_lo"]),
                       P(D["seg_hi"]), n_seg, P(D["stats_rows"]), n_stats, P(mass[l]), n, H, Hkv, dh, dt, s)
        pending_cut = None
        if focus is not None and focus.result is None and n_stats:
            # question rows are the last stats span; their mass onto each chunk span
            q0, q1 = focus.q_span
            nq = q1 - q0
            row = mass[l, n_stats - nq:n_stats, : focus.k].sum(dim=0)
            if tp is not None:  # K8a saw this rank's heads only
                row = row / tp.world
                tp.allreduce_(row)
            res = focus.tracker.push(row.cpu().numpy())
            if res is not None:
                focus.result = res
                if res.cutoff_layer < L:
                    slots = focus.cut_slots(set(res.focused))
                    if slots.size:
                        pending_cut = (slots, res.cutoff_layer)
        if record:
            lazy.q[l] = q_rot[:n_l].clone()
            lazy.lse[l] = lse[:n_l].clone()
            lazy.rows[l] = plan.rows[:n_l].copy()
            if focus is not None:  # a later cut rewrites row_slot in place
                lazy.row_slot[l] = D["row_slot"][:n_l].clone()
        if record_values:
            vtrace.append((kv_v[l], ctx[:n_l].clone(), plan.rows[:n_l].copy()))
        with tm.span("gemm", flops=2.0 * n_l * qw * d):
            if tp is None:
                N.call("cc_gemm", P(ctx), qw, P(lw["w_o"]), qw, P(hidden), d, n_l, d, qw, N.EPI_RESID_ADD, dt,
                       gemm_impl, s)
            else:
                _tp_partial_gemm(model, tp, ctx, qw, lw["w_o"], hidden, part, n_l, d, qw, dt, gemm_impl, s)
        with tm.span("rmsnorm", nbytes=n_l * d * (4 + esz)):
            N.call("cc_rmsnorm", P(hidden), P(xn), P(lw.get("mlp_norm")), n_l, d, eps, dt, s)
        if cfg.mlp == "swiglu":
            with tm.span("gemm", flops=2.0 * n_l * 2 * ff * d):
                N.call("cc_gemm", P(xn), d, P(lw["w_gu"]), d, P(act), ff, n_l, 2 * ff, d, N.EPI_SWIGLU, dt,
                       gemm_impl, s)
        else:
            with tm.span("gemm", flops=2.0 * n_l * ff * d):
                N.call("cc_gemm", P(xn), d, P(lw["w_up"]), d, P(act), ff, n_l, ff, d, N.EPI_GELU, dt, gemm_impl, s)
        with tm.span("gemm", flops=2.0 * n_l * ff * d):
            if tp is None:
                N.call("cc_gemm", P(act), ff, P(lw["w_down"]), ff, P(hidden), d, n_l, d, ff, N.EPI_RESID_ADD, dt,
                       gemm_impl, s)
            else:
                _tp_partial_gemm(model, tp, act, ff, lw["w_down"], hidden, part, n_l, d, ff, dt, gemm_impl, s)
        if pending_cut is not None:
            _apply_cut(model, plan, ws, pending_cut[0], pending_cut[1])
            focus.cut = True
            if n_stats:
                n_stats = plan.stats_rows.size
    if mass is not None and getattr(plan, "stats_cut_rows", None):
        # rows of a stats span cut by the online focus stop at the cut layer:
        # the segment-mass kernel read stale rows for them afterwards
        for rows_, depth_ in plan.stats_cut_rows:
            mass[depth_:, rows_] = 0.0
    if tp is not None and mass is not None:
        # K8a divides by the rank's own heads: global head mean = sum over ranks / world
        mass.mul_(1.0 / tp.world)
        tp.allreduce_(mass)
    return lazy, vtrace, mass


def _tp_partial_gemm(model, tp, a, lda, w, hidden, part, n_l, d, k, dt, gemm_impl, s):
    """Row-parallel projection: partial = a_local @ W_local^T on this rank,
    summed over the TP group, then hidden += sum.  bf16 with a PeerComm: the
    reduce-scatter is fused into the GEMM epilogue (P2P pushes) and the owner
    reduction + all-gather runs over peer memory (csrc/tp_peer.cu); otherwise
    an NCCL all-reduce of the partial."""
    import ctypes

    P = N.ptr
    peer = getattr(tp, "peer", None)
    if peer is not None and dt == N.BF16 and n_l <= peer.m_cap and d == peer.d:
        peer.epoch += 1
        tab = peer.table()
        addr = ctypes.addressof(tab)
        N.call("cc_tp_push_gemm", P(a), lda, P(w), lda, n_l, d, k, addr, s)
        N.call("cc_tp_reduce", addr, n_l, d, s)
        bn = 256 if peer.slice % 256 == 0 else 128
        peer.done_target += (-(-n_l // 128)) * (d // bn)
        N.call("cc_tp_wait", addr, peer.done_target, s)
        N.call("cc_add_f32", P(hidden), P(peer.local["sum"]), n_l * d, s)
        return
    if dt == N.F64:
        part[:n_l].zero_()
        N.call("cc_gemm", P(a), lda, P(w), lda, P(part), d, n_l, d, k, N.EPI_RESID_ADD, dt, gemm_impl, s)
        tp.allreduce_(part[:n_l])
        hidden[:n_l].add_(part[:n_l])
        return
    part[:n_l].zero_()
    N.call("cc_gemm", P(a), lda, P(w), lda, P(part), d, n_l, d, k, N.EPI_RESID_ADD, dt, gemm_impl, s)
    tp.allreduce_(part[:n_l])
    N.call("cc_add_f32", P(hidden), P(part), n_l * d, s)


def _payloads(model: Model, request):
    cfg = model.kcfg
    out = []
    for seg in request.segments:
        c = seg.cache
        if c is None:
            out.append(None)
            continue
        if c.n_layers != cfg.n_layers:
            raise PlanError(f"injected cache has {c.n_layers} layers, model has {cfg.n_layers}")
        if c.width != cfg.kv_width() and c.width != model.config.kv_width():
            raise ShapeError("injected cache width != kv width (d_model for MHA)")
        out.append(c.device_payload(model))
    return out


def run_prefill(model: Model, request, record_values: bool = False, record_attention="auto", stats="auto",
                first_token: bool = False, gemm_impl: int = 0, attn_impl: int = 0,
                focus_window: int | None = None) -> PrefillResult:
    import torch

    N.require_cuda()
    cfg = model.kcfg
    payloads = _payloads(model, request)
    fresh = [i for i, seg in enumerate(request.segments) if seg.cache is None]
    q0, q1 = request.question_span
    focus = None
    if focus_window is not None and len(request.segments) >= 3 and q1 > q0 and any(
            seg.cache is not None and seg.recompute is not None and np.asarray(seg.recompute).any()
            for seg in request.segments):
        focus = OnlineFocus(request, focus_window, cfg.n_layers)
        stats = True
    if stats == "auto":
        stats = bool(fresh)
    stats_segments = None
    if stats:
        stats_segments = list(request.segment_slots)
        if request.question_span[1] > request.question_span[0]:
            stats_segments.append(tuple(request.question_span))
        # only fully recomputed spans can carry stats rows (stats.py:55-65)
        ok = request.recompute_mask & (np.where(request.recompute_depth == FULL_DEPTH, cfg.n_layers,
                                                 request.recompute_depth) >= cfg.n_layers)
        stats_rows_spans = [(lo, hi) for (lo, hi) in stats_segments if hi > lo and ok[lo:hi].all()]
    plan = DevicePlan(model, request.token_ids, request.positions, request.is_pad, request.recompute_mask,
                      request.recompute_depth, request.segment_slots, payloads, request.question_span)
    if stats:
        plan.stats_segments = stats_segments
        _attach_stats_rows(model, plan, stats_rows_spans)
    if record_attention == "auto":
        record_attention = _record_default(model, plan)
    ws = _workspace(model, plan)
    lazy, vtrace, mass = execute(model, plan, ws, record=bool(record_attention), record_values=record_values,
                                 stats=bool(stats), gemm_impl=gemm_impl, attn_impl=attn_impl, focus=focus)
    extras = {"plan": plan, "ws": ws, "mass": mass, "stats_spans": stats_rows_spans if stats else None,
              "focus": None if focus is None else focus.result, "focus_cut": bool(focus is not None and focus.cut)}
    if first_token and q1 > q0:
        r = int(np.flatnonzero(plan.rows == q1 - 1)[0])
        if plan.n_act[-1] <= r:
            raise PlanError("the question's last row is not computed through every layer")
        logits, tok = _logits_rows(model, ws["hidden"][r:r + 1])
        extras["logits_last"] = logits
        extras["first_token_dev"] = tok
        # asynchronous readback into pinned memory + an event right behind
        # this request's kernels: PrefillResult.first_token waits for this
        # request only, so a server can enqueue the next request first
        host_tok = torch.empty(tok.numel(), dtype=tok.dtype, pin_memory=True)
        host_tok.copy_(tok.reshape(-1), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        extras["first_token_host"] = (host_tok, ev)
    L = cfg.n_layers
    attn = AttentionRecord(query_slots=[np.sort(plan.rows[:plan.n_act[l]]) for l in range(L)], _lazy=lazy)
    if lazy is None:
        attn._lazy = LazyAttention(model, plan, ws["k_rot"])
    depth_eff = np.where(request.recompute_depth == FULL_DEPTH, L, request.recompute_depth)
    if focus is not None and focus.cut:
        depth_eff = depth_eff.copy()
        depth_eff[plan.rows] = plan.row_depth

    def hidden_fn():
        out = torch.zeros((plan.n, cfg.d_model), dtype=torch.float64, device=model.device)
        if plan.n_rows:
            idx = torch.from_numpy(plan.rows.astype(np.int64)).to(model.device)
            out[idx] = ws["hidden"][: plan.n_rows].double()
        return out.cpu().numpy()

    res = PrefillResult(
        kv=KVCache(positions=request.positions.copy(), valid=~request.is_pad, _dev=(ws["kv_k"], ws["kv_v"])),
        attn=attn,
        question_span=request.question_span,
        computed=request.recompute_mask & (depth_eff >= L),
        active_per_layer=list(plan.n_act),
        positions=request.positions.copy(),
        hidden_fn=hidden_fn,
        extras=extras,
    )
    res.model = model
    res.request = request
    if record_values:
        res.value_trace = _ValueTrace(vtrace, plan)
    return res


def _attach_stats_rows(model, plan: DevicePlan, spans):
    """Stats rows (row indices in hidden order) for the given slot spans."""
    import torch

    pos_in_rows = np.full(plan.n, -1, np.int64)
    pos_in_rows[plan.rows] = np.arange(plan.rows.size)
    rows = [pos_in_rows[lo:hi] for lo, hi in spans]
    sr = np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32)
    plan.stats_rows = sr
    plan.stats_row_spans = spans
    plan.stats_keys = float(plan.rows[sr].astype(np.int64).sum() + sr.size)  # causal keys the K8 rows score
    segs = plan.stats_segments
    host = np.concatenate([sr, np.array([a for a, _ in segs], np.int32), np.array([b for _, b in segs], np.int32)])
    dev = torch.from_numpy(host).to(model.device)
    plan.d["stats_rows"] = dev[: sr.size]
    plan.d["seg_lo"] = dev[sr.size: sr.size + len(segs)]
    plan.d["seg_hi"] = dev[sr.size + len(segs):]


class _ValueTrace(list):
    """Per-layer (V [n, kvw], pre-projection ctx [n_act, q_width]) as numpy,
    ctx rows in ascending slot order (model.py:421-426)."""

    def __init__(self, raw, plan):
        out = []
        for l, (v, c, rows) in enumerate(raw):
            vv = v.double().cpu().numpy()
            if c is None:
                out.append((vv, np.zeros((0, v.shape[-1]))))
                continue
            order = np.argsort(rows, kind="stable")
            out.append((vv, c.double().cpu().numpy()[order]))
        super().__init__(out)


def _logits_rows(model: Model, rows_dev):
    import torch

    cfg = model.config
    m = rows_dev.shape[0]
    logits = torch.empty((m, cfg.vocab_size), dtype=model.hidden_dtype, device=model.device)
    tok = torch.empty((m,), dtype=torch.int32, device=model.device)
    N.call("cc_logits_argmax", N.ptr(rows_dev.contiguous()), N.ptr(model.w.get("final_norm")), cfg.rms_eps,
           N.ptr(model.w["unembed_t"]), N.ptr(logits), N.ptr(tok), m, cfg.d_model, cfg.vocab_size, model.dtype_code,
           N.stream_ptr())
    return logits, tok


def logits_device(model: Model, hidden_rows):
    """Model.logits on the GPU (model.py:94-95): returns (logits, argmax)."""
    import torch

    N.require_cuda()
    h = np.atleast_2d(np.asarray(hidden_rows, dtype=np.float64))
    if h.shape[1] != model.config.d_model:
        raise ShapeError("hidden rows width != d_model")
    outs, toks = [], []
    for i in range(0, h.shape[0], 8):
        rows = torch.from_numpy(h[i:i + 8]).to(model.device, model.hidden_dtype)
        lg, tk = _logits_rows(model, rows)
        outs.append(lg.double().cpu().numpy())
        toks.append(tk.cpu().numpy())
    return np.concatenate(outs), np.concatenate(toks)


def extract_rows(result: PrefillResult, start: int, stop: int, source_prefix=()) -> ChunkCache:
    """K10: request KV rows [start, stop) -> fresh pool blocks of a new cache."""
    model = result.model
    cfg = model.kcfg
    kv_k, kv_v = result.kv._dev if result.kv._dev is not None else (None, None)
    n = stop - start
    if n <= 0:
        raise PlanError("empty row range")
    if kv_k is None:
        keys, values = result.kv.slice_rows(start, stop)
        return ChunkCache(keys=keys, values=values, n_tokens=n, source_prefix=source_prefix)
    pool = model.pool
    nb = -(-n // BLOCK)
    blocks = pool.alloc(nb)
    import torch

    bdev = torch.from_numpy(blocks).to(model.device)
    N.call("cc_extract_to_pool", N.ptr(kv_k), N.ptr(kv_v), kv_k.stride(0), cfg.n_layers, start, n, N.ptr(bdev), nb,
           N.ptr(pool.storage), pool.layer_stride, pool.block_stride, cfg.kv_width(), model.dtype_code, N.stream_ptr())
    return ChunkCache(n_tokens=n, source_prefix=source_prefix, _payload=_Payload(pool, blocks, n))


class DecodeSession:
    """Greedy decode on the device (model.py:445-484).

    The request KV is copied once into capacity buffers [L][n0 + max_steps]
    (position-free ``kv_k``/``kv_v`` + ``k_rot`` rotated at the key positions,
    pads at position 0 as in the reference, :466); every step then runs the
    per-layer pipeline for the single new row entirely on the stream: the
    token id never leaves the device (argmax -> embedding), the new K/V row is
    scattered in place (cc_rope_scatter_qkv), attention is the split-KV
    cc_decode_attention (bf16) and the projections are weight-streaming
    GEMVs (cc_gemm routes M = 1 there).  Tokens are read back once."""

    def __init__(self, model: Model, kv: KVCache, max_steps: int):
        import torch

        cfg = model.kcfg
        self.model, self.kv, self.steps = model, kv, int(max_steps)
        L, kvw = cfg.n_layers, cfg.kv_width()
        dev, T = model.device, model.torch_dtype
        n0 = kv.n_slots
        cap = n0 + self.steps
        self.n0, self.cap = n0, cap
        valid = np.asarray(kv.valid, bool)
        positions = np.asarray(kv.positions, np.int64)
        if not valid.any():
            raise PlanError("decode needs at least one valid KV row")
        self.next_pos = int(positions[valid].max()) + 1
        key_pos = np.where(valid, positions, 0)
        pos_all = np.concatenate([key_pos, self.next_pos + np.arange(self.steps)]).astype(np.int32)
        slots = (n0 + np.arange(self.steps)).astype(np.int32)
        pad = np.zeros(-(-cap // 16) * 16, np.uint8)
        pad[:n0] = ~valid
        self.has_pad = bool((~valid).any())
        self.kv_k = torch.empty((L, cap, kvw), dtype=T, device=dev)
        self.kv_v = torch.empty((L, cap, kvw), dtype=T, device=dev)
        self.k_rot = torch.empty((L, cap, kvw), dtype=T, device=dev)
        if n0:
            if kv._dev is not None:
                self.kv_k[:, :n0].copy_(kv._dev[0][:, :n0])
                self.kv_v[:, :n0].copy_(kv._dev[1][:, :n0])
            else:
                self.kv_k[:, :n0].copy_(torch.from_numpy(np.stack(kv.keys)).to(dev, T))
                self.kv_v[:, :n0].copy_(torch.from_numpy(np.stack(kv.values)).to(dev, T))
        self.pos = torch.from_numpy(pos_all).to(dev)
        self.slots = torch.from_numpy(slots).to(dev)
        self.pad = torch.from_numpy(pad).to(dev)
        self.rope = model.rope_table(self.next_pos + self.steps)
        if n0:
            N.call("cc_rope_rows", N.ptr(self.kv_k), N.ptr(self.k_rot), L * cap, cap, kvw, N.ptr(self.pos),
                   N.ptr(self.rope), cfg.head_dim(), model.dtype_code, N.stream_ptr())
        d, q, ff = cfg.d_model, cfg.q_width(), cfg.ff_dim()
        Hd = model.hidden_dtype
        e = torch.empty
        self.hidden = e((1, d), dtype=Hd, device=dev)
        self.part = e((1, d), dtype=Hd, device=dev) if (model.tp is not None and model.tp.world > 1) else None
        self.xn = e((1, d), dtype=T, device=dev)
        self.qkv = e((1, q + 2 * kvw), dtype=T, device=dev)
        self.q_rot = e((1, q), dtype=T, device=dev)
        self.ctx = e((1, q), dtype=T, device=dev)
        self.act = e((1, ff), dtype=T, device=dev)
        self.lse = e((1, cfg.n_heads), dtype=Hd, device=dev)
        self.tokens = torch.zeros((self.steps + 1,), dtype=torch.int32, device=dev)
        self.logits = e((1, model.config.vocab_size), dtype=Hd, device=dev)
        self.state = torch.zeros((4,), dtype=torch.int32, device=dev)
        self.cur = torch.zeros((1,), dtype=torch.int32, device=dev)
        tp = model.tp is not None and model.tp.world > 1
        self.fast_attn = (model.dtype_code == N.BF16 and cfg.head_dim() == 128
                          and cfg.n_heads // cfg.kv_heads() in (1, 2, 4, 8))
        self.graphable = self.fast_attn and not tp
        # bf16: RoPE + append + split-KV attention + combine in one launch per layer
        self.fused_attn = self.fast_attn and cap <= 131072 and os.environ.get("CCB_DECODE_FUSED", "1") != "0"
        # bf16: fused RMSNorm + weight-streaming GEMV (cc_gemv_rmsnorm) when eligible
        self.fused_norm = (model.dtype_code == N.BF16 and cfg.d_model % 8 == 0
                           and cfg.d_model * 2 <= 96 * 1024 and (cfg.mlp != "swiglu" or (2 * cfg.ff_dim()) % 128 == 0))
        self.graph = None
        self.replay_events = None
        # programmatic dependent launch: the streaming GEMVs fill their weight
        # rings before griddepcontrol.wait, so each one's first ~100 KiB per SM
        # load while its predecessor runs (with the unfused chain PDL measured
        # slower: parked dependents only cut the running GEMV's occupancy)
        self.pdl = self.fused_attn and os.environ.get("CCB_DECODE_PDL", "1") != "0"

    def _argmax(self, rows, out_ptr):
        m = self.model
        cfg = m.config
        N.call("cc_logits_argmax", N.ptr(rows), N.ptr(m.w.get("final_norm")), cfg.rms_eps, N.ptr(m.w["unembed_t"]),
               N.ptr(self.logits), out_ptr, 1, cfg.d_model, cfg.vocab_size, m.dtype_code, N.stream_ptr())

    def _layers(self, tok_ptr, slot_ptr, pos_ptr, n_keys):
        """One token through every layer.  ``n_keys`` is the live key count
        (eager) or None (graph mode: read from ``state[3]`` on the device)."""
        m = self.model
        cfg = m.kcfg
        tp = m.tp if (m.tp is not None and m.tp.world > 1) else None
        P, s, dt = N.ptr, N.stream_ptr(), m.dtype_code
        H, Hkv, dh, d = cfg.n_heads, cfg.kv_heads(), cfg.head_dim(), cfg.d_model
        qw, kvw, ff = cfg.q_width(), cfg.kv_width(), cfg.ff_dim()
        pad = P(self.pad) if self.has_pad else None
        hid = self.hidden
        N.call("cc_embed_rows", P(m.w["embed"]), tok_ptr, P(hid), 1, d, dt, s)
        for l in range(cfg.n_layers):
            lw = m.w["layers"][l]
            if self.fused_norm:  # RMSNorm in the GEMV prologue
                N.call("cc_gemv_rmsnorm", P(hid), d, P(lw.get("attn_norm")), cfg.rms_eps, P(lw["w_qkv"]), d,
                       P(self.qkv), qw + 2 * kvw, 1, qw + 2 * kvw, d, N.EPI_STORE, s)
            else:
                N.call("cc_rmsnorm", P(hid), P(self.xn), P(lw.get("attn_norm")), 1, d, cfg.rms_eps, dt, s)
                N.call("cc_gemm", P(self.xn), d, P(lw["w_qkv"]), d, P(self.qkv), qw + 2 * kvw, 1, qw + 2 * kvw, d,
                       N.EPI_STORE, dt, 0, s)
            if self.fused_attn:
                N.call("cc_decode_attention_qkv", P(self.qkv), slot_ptr, pos_ptr, P(self.rope), P(self.kv_k[l]),
                       P(self.kv_v[l]), P(self.k_rot[l]), pad, P(self.ctx), P(self.lse), n_keys or 0,
                       P(self.state[3:4]) if n_keys is None else None, self.cap, H, Hkv, dh, s)
            else:
                N.call("cc_rope_scatter_qkv", P(self.qkv), qw + 2 * kvw, 1, slot_ptr, pos_ptr, P(self.rope),
                       P(self.q_rot), P(self.kv_k[l]), P(self.kv_v[l]), P(self.k_rot[l]), H, Hkv, dh, dt, s)
                if n_keys is None:
                    N.call("cc_decode_attention_dev", P(self.q_rot), P(self.k_rot[l]), P(self.kv_v[l]), pad,
                           P(self.ctx), P(self.lse), P(self.state[3:4]), self.cap, H, Hkv, dh, s)
                elif self.fast_attn:
                    N.call("cc_decode_attention", P(self.q_rot), P(self.k_rot[l]), P(self.kv_v[l]), pad,
                           P(self.ctx), P(self.lse), n_keys, H, Hkv, dh, s)
                else:
                    N.call("cc_attention", P(self.q_rot), P(self.k_rot[l]), P(self.kv_v[l]), slot_ptr, pad,
                           P(self.ctx), P(self.lse), 1, n_keys, H, Hkv, dh, dt, 0, s)
            if tp is None:
                N.call("cc_gemm", P(self.ctx), qw, P(lw["w_o"]), qw, P(hid), d, 1, d, qw, N.EPI_RESID_ADD, dt, 0, s)
            else:
                _tp_partial_gemm(m, tp, self.ctx, qw, lw["w_o"], hid, self.part, 1, d, qw, dt, 0, s)
            if self.fused_norm:
                w_in, n_in, epi = (lw["w_gu"], 2 * ff, N.EPI_SWIGLU) if cfg.mlp == "swiglu" else (
                    lw["w_up"], ff, N.EPI_GELU)
                N.call("cc_gemv_rmsnorm", P(hid), d, P(lw.get("mlp_norm")), cfg.rms_eps, P(w_in), d, P(self.act), ff,
                       1, n_in, d, epi, s)
            else:
                N.call("cc_rmsnorm", P(hid), P(self.xn), P(lw.get("mlp_norm")), 1, d, cfg.rms_eps, dt, s)
                if cfg.mlp == "swiglu":
                    N.call("cc_gemm", P(self.xn), d, P(lw["w_gu"]), d, P(self.act), ff, 1, 2 * ff, d, N.EPI_SWIGLU,
                           dt, 0, s)
                else:
                    N.call("cc_gemm", P(self.xn), d, P(lw["w_up"]), d, P(self.act), ff, 1, ff, d, N.EPI_GELU, dt, 0,
                           s)
            if tp is None:
                N.call("cc_gemm", P(self.act), ff, P(lw["w_down"]), ff, P(hid), d, 1, d, ff, N.EPI_RESID_ADD, dt,
                       0, s)
            else:
                _tp_partial_gemm(m, tp, self.act, ff, lw["w_down"], hid, self.part, 1, d, ff, dt, 0, s)

    def _graph_step(self):
        """One decode step driven entirely by device state (graph-capturable):
        embed(cur) -> layers at (state slot, pos, live keys) -> argmax -> cur
        -> advance (tokens[count] = cur; count, slot, pos, keys += 1)."""
        P = N.ptr
        self._layers(P(self.cur), P(self.state[1:2]), P(self.state[2:3]), None)
        self._argmax(self.hidden, P(self.cur))
        N.call("cc_decode_advance", P(self.state), P(self.cur), P(self.tokens), N.stream_ptr())

    def run(self, last_hidden_dev) -> None:
        """Enqueue all steps.  bf16 / d_head 128 without TP: step 0 runs
        eagerly on a private stream (warms every kernel), the step body is
        captured once as a CUDA graph and replayed for the remaining steps —
        no per-token host work.  Otherwise every step is launched eagerly."""
        import torch

        prev_pdl = N.lib().cc_set_pdl(1 if self.pdl else 0)
        try:
            self._run(last_hidden_dev)
        finally:
            N.lib().cc_set_pdl(prev_pdl)

    def _run(self, last_hidden_dev) -> None:
        import torch

        P = N.ptr
        if not self.graphable:
            self._argmax(last_hidden_dev, P(self.tokens[0:1]))
            for step in range(self.steps):
                slot = self.n0 + step
                self._layers(P(self.tokens[step:step + 1]), P(self.slots[step:step + 1]), P(self.pos[slot:slot + 1]),
                             slot + 1)
                if step + 1 < self.steps:
                    self._argmax(self.hidden, P(self.tokens[step + 1:step + 2]))
            return
        # state = [count, slot, position, live keys], primed so the first advance
        # lands on (1, n0, next_pos, n0 + 1)
        init = torch.tensor([0, self.n0 - 1, self.next_pos - 1, self.n0], dtype=torch.int32)
        cs = torch.cuda.Stream(device=self.model.device)
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            self.state.copy_(init, non_blocking=False)
            self._argmax(last_hidden_dev, P(self.cur))
            N.call("cc_decode_advance", P(self.state), P(self.cur), P(self.tokens), N.stream_ptr())
            self._graph_step()  # step 0, eager
        if self.steps > 1:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                self._graph_step()
            self.graph = g
            self.replay_events = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            with torch.cuda.stream(cs):
                self.replay_events[0].record(cs)
                for _ in range(self.steps - 1):
                    g.replay()
                self.replay_events[1].record(cs)
        torch.cuda.current_stream().wait_stream(cs)
        self.stream = cs

    def finish(self) -> list:
        """Read the tokens back and extend the caller's KVCache in place
        (kv.append_token semantics: position-free rows, positions next_pos..)."""
        toks = [int(t) for t in self.tokens[: self.steps].cpu().numpy()]
        kv = self.kv
        new_pos = self.next_pos + np.arange(self.steps)
        kv._keys = None
        kv._values = None
        kv._dev = (self.kv_k, self.kv_v)
        kv.positions = np.concatenate([np.asarray(kv.positions, np.int64), new_pos])
        kv.valid = np.concatenate([np.asarray(kv.valid, bool), np.ones(self.steps, bool)])
        return toks


def run_decode(model: Model, kv: KVCache, last_hidden, max_steps: int) -> list:
    """Greedy decode (model.py:445-484) on the device: see DecodeSession."""
    import torch

    if max_steps <= 0:
        return []
    N.require_cuda()
    sess = DecodeSession(model, kv, max_steps)
    if isinstance(last_hidden, torch.Tensor):
        h = last_hidden.reshape(1, -1).to(model.device, model.hidden_dtype)
    else:
        h = torch.from_numpy(np.asarray(last_hidden, dtype=np.float64).reshape(1, -1)).to(model.device,
                                                                                      model.hidden_dtype)
    if h.shape[1] != model.config.d_model:
        raise ShapeError("last_hidden width != d_model")
    sess.run(h.contiguous())
    return sess.finish()
