"""Inter/intra attention aggregates and per-token contextualisation scores
(cachecraft/stats.py:1-176, harness.py:331-354).

Two paths:
  * the creation-time hot path (``creation_stats``, ``question_stream``):
    kernel K8a (``cc_segment_mass``) reduces head-mean attention mass per
    (query row, key segment) during prefill without materialising weights,
    and kernel K8b (``cc_chunk_stats``) folds those masses into inter / intra
    / token scores with deterministic fixed-order sums;
  * the reference's analysis API (``inter``, ``intra``, ``compute_stats`` ...)
    over an ``AttentionRecord``: weights are materialised on the GPU
    (``cc_attention_probs``) and reduced there.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ArgumentError, PlanError
from .model import AttentionRecord
from .scoring import PrefixContext


@dataclass(frozen=True)
class ChunkSpan:
    """Slot range of one chunk's real tokens (stats.py:22-34)."""

    chunk_id: object
    start: int
    length: int

    @property
    def stop(self) -> int:
        return self.start + self.length

    def slots(self) -> np.ndarray:
        return np.arange(self.start, self.stop)


def spans_from_lengths(chunk_ids, lengths, slot_lengths=None) -> list:
    """Spans of chunks laid out back to back (stats.py:37-52)."""
    slot_lengths = lengths if slot_lengths is None else slot_lengths
    out, cursor = [], 0
    for cid, n_real, n_slots in zip(chunk_ids, lengths, slot_lengths):
        if n_real < 1 or n_slots < n_real:
            raise ArgumentError(f"bad span lengths for chunk {cid}: {n_real}/{n_slots}")
        out.append(ChunkSpan(chunk_id=cid, start=cursor, length=n_real))
        cursor += n_slots
    return out


# ---------------------------------------------------------------------------
# analysis API over an AttentionRecord (GPU reductions)
# ---------------------------------------------------------------------------


def _head_mean_dev(attn: AttentionRecord, layer: int):
    import torch

    cache = attn.__dict__.setdefault("_hm_dev", {})
    if layer not in cache:
        if attn._weights is None and attn._lazy is not None and attn._lazy.q:
            w = torch.from_numpy(attn._lazy.materialize(layer))
        else:
            w = torch.from_numpy(np.asarray(attn.weights[layer], dtype=np.float64))
        cache[layer] = w.to("cuda").mean(dim=0)
    return cache[layer]


def _rows_for(attn: AttentionRecord, layer: int, span: ChunkSpan) -> np.ndarray:
    lookup = attn.row_lookup(layer)
    rows = []
    for slot in range(span.start, span.stop):
        if slot not in lookup:
            raise ArgumentError(f"attention rows missing for slot {slot} at layer {layer}; "
                                "stats need fully computed chunks")
        rows.append(lookup[slot])
    return np.asarray(rows, dtype=np.int64)


def _block_sum(attn, layer, rows, c0, c1, lower=False, diag=False) -> float:
    import torch

    a = _head_mean_dev(attn, layer)
    r = torch.from_numpy(rows).to(a.device)
    blk = a.index_select(0, r)[:, c0:c1]
    if diag:
        return float(torch.diagonal(blk).sum().item())
    if lower:
        blk = torch.tril(blk, diagonal=-1)
    return float(blk.sum().item())


def inter(attn: AttentionRecord, spans, i: int, j: int, layer: int) -> float:
    """Head-mean mass from chunk j's queries onto chunk i's keys (stats.py:68-75)."""
    if i >= j:
        raise ArgumentError(f"inter needs i < j in span order, got {i} >= {j}")
    N.require_cuda()
    return _block_sum(attn, layer, _rows_for(attn, layer, spans[j]), spans[i].start, spans[i].stop)


def intra(attn: AttentionRecord, spans, i: int, layer: int) -> float:
    """Strictly-below-diagonal mass inside chunk i (stats.py:78-84)."""
    N.require_cuda()
    sp = spans[i]
    return _block_sum(attn, layer, _rows_for(attn, layer, sp), sp.start, sp.stop, lower=True)


def diagonal_mass(attn: AttentionRecord, spans, i: int, layer: int) -> float:
    N.require_cuda()
    sp = spans[i]
    return _block_sum(attn, layer, _rows_for(attn, layer, sp), sp.start, sp.stop, diag=True)


def token_inter_scores(attn: AttentionRecord, spans, i: int) -> np.ndarray:
    """Per-token mass onto all earlier chunks, summed over layers (stats.py:94-106)."""
    import torch

    sp = spans[i]
    if i == 0:
        return np.zeros(sp.length)
    N.require_cuda()
    cols = torch.from_numpy(np.concatenate([spans[j].slots() for j in range(i)])).to("cuda")
    acc = None
    for layer in range(attn.n_layers):
        a = _head_mean_dev(attn, layer)
        r = torch.from_numpy(_rows_for(attn, layer, sp)).to(a.device)
        part = a.index_select(0, r).index_select(1, cols).sum(dim=1)
        acc = part if acc is None else acc + part
    return acc.cpu().numpy()


@dataclass
class AttentionStats:
    spans: list
    inter_table: dict
    intra_table: dict
    diag_table: dict
    token_inter: dict
    n_layers: int

    def inter_layer_sum(self, i: int, j: int) -> float:
        return float(self.inter_table[(i, j)].sum())

    def prefix_weights(self, i: int) -> dict:
        return {self.spans[j].chunk_id: self.inter_layer_sum(j, i) for j in range(i)}


def compute_stats(attn: AttentionRecord, spans) -> AttentionStats:
    L = attn.n_layers
    it, ia, dg, tk = {}, {}, {}, {}
    for i in range(len(spans)):
        ia[i] = np.array([intra(attn, spans, i, l) for l in range(L)])
        dg[i] = np.array([diagonal_mass(attn, spans, i, l) for l in range(L)])
        tk[i] = token_inter_scores(attn, spans, i)
        for j in range(i):
            it[(j, i)] = np.array([inter(attn, spans, j, i, l) for l in range(L)])
    return AttentionStats(spans=list(spans), inter_table=it, intra_table=ia, diag_table=dg, token_inter=tk, n_layers=L)


def context_ratios(stats: AttentionStats, i: int) -> tuple:
    """Layer means of the normalised outside/self sums (stats.py:150-157)."""
    sp = stats.spans[i]
    a = np.zeros(stats.n_layers)
    for j in range(i):
        a += stats.inter_table[(j, i)] / (sp.length * stats.spans[j].length)
    b = stats.intra_table[i] / sp.length**2
    return float(a.mean()), float(b.mean())


def question_inter_stream(attn: AttentionRecord, spans, question_span) -> np.ndarray:
    """[L, k] question->chunk mass per layer (stats.py:160-176)."""
    import torch

    q0, q1 = question_span
    L, k = attn.n_layers, len(spans)
    out = np.zeros((L, k))
    if q1 == q0:
        return out
    N.require_cuda()
    for layer in range(L):
        lookup = attn.row_lookup(layer)
        rows = np.asarray([lookup[s] for s in range(q0, q1) if s in lookup], dtype=np.int64)
        if rows.size == 0:
            continue
        a = _head_mean_dev(attn, layer)
        blk = a.index_select(0, torch.from_numpy(rows).to(a.device))
        for i, sp in enumerate(spans):
            out[layer, i] = float(blk[:, sp.start:sp.stop].sum().item())
    return out


# ---------------------------------------------------------------------------
# creation-time hot path: K8a masses (recorded during prefill) -> K8b
# ---------------------------------------------------------------------------


def _k8b(result, chunk_indices):
    import torch

    ex = result.extras
    mass, plan = ex.get("mass"), ex.get("plan")
    if mass is None:
        raise PlanError("prefill ran without stats; call prefill(..., stats=True)")
    spans = plan.stats_row_spans
    seg_index = {s: k for k, s in enumerate(plan.stats_segments)}
    row0, lens, seg_of, tok_off = [], [], [], []
    start = {}
    cur = 0
    for sp in spans:
        start[sp] = cur
        cur += sp[1] - sp[0]
    toff = 0
    for i in chunk_indices:
        sp = tuple(result.request.segment_slots[i])
        if sp not in start:
            raise ArgumentError(f"chunk {i} is not fully recomputed; stats need fresh chunks")
        row0.append(start[sp])
        lens.append(sp[1] - sp[0])
        seg_of.append(seg_index[sp])
        tok_off.append(toff)
        toff += sp[1] - sp[0]
    L = result.model.config.n_layers
    n_seg = len(plan.stats_segments)
    n_rows = mass.shape[1]
    C = len(chunk_indices)
    dev = mass.device
    meta = torch.from_numpy(np.array(row0 + lens + seg_of + tok_off, dtype=np.int32)).to(dev)
    inter_t = torch.empty((C, L, n_seg), dtype=torch.float64, device=dev)
    intra_t = torch.empty((C, L), dtype=torch.float64, device=dev)
    tok_t = torch.empty((max(toff, 1),), dtype=torch.float64, device=dev)
    N.call("cc_chunk_stats", N.ptr(mass), L, n_rows, n_seg, N.ptr(meta[0:C]), N.ptr(meta[C:2 * C]),
           N.ptr(meta[2 * C:3 * C]), N.ptr(meta[3 * C:4 * C]), C, N.ptr(inter_t), N.ptr(intra_t), N.ptr(tok_t),
           N.stream_ptr())
    return inter_t.cpu().numpy(), intra_t.cpu().numpy(), tok_t, tok_off, lens


def creation_stats(result, chunk_ids, chunk_indices) -> dict:
    """Creation-time metadata of freshly computed chunks (harness.py:331-354):
    index -> (PrefixContext, a_bar, b_bar, token_scores [device float64]).
    ``chunk_ids`` names every request segment (for the prefix)."""
    if not chunk_indices:
        return {}
    inter_h, intra_h, tok_dev, tok_off, lens = _k8b(result, list(chunk_indices))
    slots = result.request.segment_slots
    out = {}
    for c, i in enumerate(chunk_indices):
        li = lens[c]
        L = inter_h.shape[1]
        a_l = np.zeros(L)
        wsum: dict = {}
        for j in range(i):
            lj = slots[j][1] - slots[j][0]
            il = inter_h[c, :, j]
            a_l += il / (li * lj)
            wsum[chunk_ids[j]] = wsum.get(chunk_ids[j], 0.0) + float(il.sum())
        b_l = intra_h[c] / li**2
        ids = list(dict.fromkeys(chunk_ids[:i]))
        prefix = PrefixContext(chunk_ids=tuple(ids), weights=tuple(wsum[x] for x in ids))
        out[i] = (prefix, float(a_l.mean()), float(b_l.mean()), tok_dev[tok_off[c]: tok_off[c] + li])
    return out


def question_stream(result) -> np.ndarray:
    """[L, k] question->chunk mass from the K8a masses (stats.py:160-176)."""
    ex = result.extras
    mass, plan = ex.get("mass"), ex.get("plan")
    if mass is None:
        raise PlanError("prefill ran without stats; call prefill(..., stats=True)")
    q = tuple(result.request.question_span)
    k = len(result.request.segment_slots)
    L = result.model.config.n_layers
    if q[1] == q[0] or q not in plan.stats_row_spans:
        return np.zeros((L, k))
    off = 0
    for sp in plan.stats_row_spans:
        if sp == q:
            break
        off += sp[1] - sp[0]
    m = mass[:, off: off + q[1] - q[0], :k].sum(dim=1)
    return m.cpu().numpy()
