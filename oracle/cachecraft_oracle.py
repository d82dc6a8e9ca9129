"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference Cache-Craft chunk-cache fix-up prefill
(``/root/reference/pkg/src/cachecraft``), extended with the optional Llama-3
architecture knobs (GQA, SwiGLU, weighted RMSNorm, custom eps / RoPE base) so it
can check the B200 engine at Llama shapes too.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this module, and only as the CHECKER (or
as the timed CPU baseline).  The product package ``paper_2502_15734_b200``
never imports it; there is no CPU fallback in the product.

Pinning: ``tests/golden/make_golden.py`` imports the unmodified reference in the
build container and writes fixtures under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this module against every fixture
(reference-architecture mode: agreement to ~1e-12).  Each function names the
reference file:line it restates.  Citations are relative to
``/root/reference/pkg/src/cachecraft/``.

Everything here is float64 / int64, like the reference.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

FULL_DEPTH = -1  # model.py:32


# --------------------------------------------------------------------------
# configuration and weights  (model.py:36-118)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class OracleConfig:
    """Shape of the oracle model.  Defaults reproduce ``ModelConfig()``
    (model.py:43-49); the extra knobs default to the reference architecture
    (MHA, GELU-tanh FFN of width 4d, weightless RMSNorm eps 1e-6)."""

    n_layers: int = 4
    n_heads: int = 4
    d_model: int = 64
    d_head: int | None = None
    vocab_size: int = 256
    rpe_base: float = 10000.0
    seed: int = 0
    n_kv_heads: int | None = None
    d_ff: int | None = None
    mlp: str = "gelu_tanh"  # or "swiglu"
    norm_weight: bool = False
    rms_eps: float = 1e-6

    @property
    def dh(self) -> int:
        return self.d_model // self.n_heads if self.d_head is None else self.d_head

    @property
    def hkv(self) -> int:
        return self.n_heads if self.n_kv_heads is None else self.n_kv_heads

    @property
    def ff(self) -> int:
        return 4 * self.d_model if self.d_ff is None else self.d_ff

    @property
    def kv_width(self) -> int:
        return self.hkv * self.dh


def draw_weights(cfg: OracleConfig) -> dict:
    """Seeded weight stream, same draw order as build_model (model.py:103-116):
    embed, unembed, then per layer wq, wk, wv, wo, [w_gate,] w_up, w_down.
    Weights are [in, out] and applied as x @ W."""
    g = np.random.default_rng(cfg.seed)
    d, q_w, kv_w, ff = cfg.d_model, cfg.n_heads * cfg.dh, cfg.kv_width, cfg.ff

    def normal(rows, cols, fan_in=None):
        m = g.standard_normal((rows, cols))
        return m if fan_in is None else m / np.sqrt(fan_in)

    out = {"embed": normal(cfg.vocab_size, d), "unembed": normal(d, cfg.vocab_size, d), "layers": []}
    for _ in range(cfg.n_layers):
        lw = {
            "wq": normal(d, q_w, d),
            "wk": normal(d, kv_w, d),
            "wv": normal(d, kv_w, d),
            "wo": normal(q_w, d, q_w),
        }
        if cfg.mlp == "swiglu":
            lw["w_gate"] = normal(d, ff, d)
        lw["w_up"] = normal(d, ff, d)
        lw["w_down"] = normal(ff, d, ff)
        lw["attn_norm"] = np.ones(d)
        lw["mlp_norm"] = np.ones(d)
        out["layers"].append(lw)
    out["final_norm"] = np.ones(d)
    return out


def weight_bytes(w: dict) -> bytes:
    """Concatenated weight bytes in draw order (model.py:87-92)."""
    parts = [w["embed"].tobytes(), w["unembed"].tobytes()]
    for lw in w["layers"]:
        for name in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"):
            if name in lw:
                parts.append(lw[name].tobytes())
    return b"".join(parts)


def rmsnorm(x, eps=1e-6, weight=None):
    """model.py:121-122 (weight is the Llama extension; None = reference)."""
    y = x / np.sqrt(np.mean(np.square(x), axis=-1, keepdims=True) + eps)
    return y if weight is None else y * weight


def gelu_tanh(x):
    """model.py:125-126."""
    return 0.5 * x * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (x + 0.044715 * x**3)))


def silu(x):
    return x / (1.0 + np.exp(-x))


# --------------------------------------------------------------------------
# rotary embedding  (rpe.py:19-59)
# --------------------------------------------------------------------------


def rope(vectors, positions, base=10000.0, d_head=None, sign=1.0):
    """Half-split pairwise rotation (rpe.py:19-44): component j of a head's
    first half pairs with component j of its second half at angle
    sign * pos * base**(-2j/d_head)."""
    v = np.asarray(vectors, dtype=np.float64)
    n, width = v.shape
    dh = width if d_head is None else d_head
    half = dh // 2
    inv_freq = base ** (-2.0 * np.arange(half) / dh)
    ang = sign * np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    heads = v.reshape(n, width // dh, 2, half)
    a, b = heads[:, :, 0, :], heads[:, :, 1, :]
    out = np.stack([a * c - b * s, a * s + b * c], axis=2)
    return out.reshape(n, width)


# --------------------------------------------------------------------------
# request layout  (model.py:193-262)
# --------------------------------------------------------------------------


def layout(segments, question) -> dict:
    """Slot layout of a request.  ``segments`` is a list of dicts with keys
    tokens, n_slots (None for fresh text), recompute (bool[n_tok] or None),
    depth (int[n_tok] or None).  Mirrors PrefillRequest.__post_init__:
    pads trail cached rows, consume no position (-1), are never recomputed;
    fresh text and the question are always recomputed at full depth."""
    tok, pos, pad, msk, dep, spans = [], [], [], [], [], []
    slot, p = 0, 0
    for seg in segments:
        t = np.asarray(seg["tokens"], dtype=np.int64)
        nt = t.size
        ns = nt if seg.get("n_slots") is None else int(seg["n_slots"])
        m = np.zeros(ns, dtype=bool)
        d = np.zeros(ns, dtype=np.int64)
        if seg.get("n_slots") is None:  # fresh text
            m[:] = True
            d[:] = FULL_DEPTH
        else:
            if seg.get("recompute") is not None:
                m[:nt] = np.asarray(seg["recompute"], dtype=bool)
            if seg.get("depth") is not None:
                d[:nt] = np.asarray(seg["depth"], dtype=np.int64)
            else:
                d[:nt] = FULL_DEPTH
            d[:nt][~m[:nt]] = 0
        ids = np.zeros(ns, dtype=np.int64)
        ids[:nt] = t
        sp = np.full(ns, -1, dtype=np.int64)
        sp[:nt] = p + np.arange(nt)
        pd = np.zeros(ns, dtype=bool)
        pd[nt:] = True
        tok.append(ids), pos.append(sp), pad.append(pd), msk.append(m), dep.append(d)
        spans.append((slot, slot + nt))
        slot += ns
        p += nt
    q = np.asarray(question, dtype=np.int64)
    qspan = (slot, slot + q.size)
    if q.size:
        tok.append(q)
        pos.append(p + np.arange(q.size))
        pad.append(np.zeros(q.size, dtype=bool))
        msk.append(np.ones(q.size, dtype=bool))
        dep.append(np.full(q.size, FULL_DEPTH, dtype=np.int64))
    return {
        "token_ids": np.concatenate(tok),
        "positions": np.concatenate(pos),
        "is_pad": np.concatenate(pad),
        "mask": np.concatenate(msk),
        "depth": np.concatenate(dep),
        "segment_slots": spans,
        "question_span": qspan,
    }


# --------------------------------------------------------------------------
# partial prefill  (model.py:348-442)
# --------------------------------------------------------------------------


def prefill(w: dict, cfg: OracleConfig, lay: dict, caches, keep_weights=True, layers=None, tp=None,
            sample_rows=None) -> dict:
    """Partial prefill with injected position-free caches.

    ``caches`` is a list aligned with the segments: None for fresh text, else
    (keys, values) with keys[l] / values[l] of shape [n_slots, kv_width].
    Per layer (model.py:382-429): active = mask & depth > l; K/V start as the
    injected rows (zeros elsewhere); active rows get fresh q/k/v from the
    normed hidden state (cache repair); all keys are rotated at their slot
    position (0 at pads); a query sees the non-pad keys at positions <= its
    own; the residual MLP follows.  ``layers`` optionally limits the run to
    the first ``layers`` layers (bench CPU-baseline sampling).

    ``tp`` (test of the multi-GPU partition) = {"q": slice, "kv": slice,
    "ff": slice, "allreduce": fn}: this call computes one tensor-parallel
    rank — its query/kv head columns and MLP columns — and ``allreduce``
    sums the o_proj and down_proj partial outputs over the ranks before the
    residual adds (the only two reductions of a layer, model.py:417, :419).

    ``sample_rows`` (memory bound for the long-prompt parity tests): at the
    LAST layer run, K/V are still projected for every active row, but the
    attention, o_proj and MLP are evaluated only for the active rows whose
    slot is in ``sample_rows`` (each row's output depends on its own
    attention row only, so those rows are exact); other rows' hidden state
    is left at its input value at that layer.
    """
    L = cfg.n_layers if layers is None else layers
    H, Hkv, dh = cfg.n_heads, cfg.hkv, cfg.dh
    qc, kc, fc = (slice(None), slice(None), slice(None)) if tp is None else (tp["q"], tp["kv"], tp["ff"])
    if tp is not None:
        H = (qc.stop - qc.start) // dh
        Hkv = (kc.stop - kc.start) // dh
    kvw = Hkv * dh
    group = H // Hkv
    reduce = (lambda a: a) if tp is None else tp["allreduce"]
    n = lay["token_ids"].size
    d = cfg.d_model
    mask, pos, pad = lay["mask"], lay["positions"], lay["is_pad"]
    depth = np.where(lay["depth"] == FULL_DEPTH, cfg.n_layers, lay["depth"])
    hidden = np.zeros((n, d))
    hidden[mask] = w["embed"][lay["token_ids"][mask]]
    key_pos = np.where(pad, 0, pos)
    keys_out, vals_out, attn_w, attn_rows, active = [], [], [], [], []
    nw = cfg.norm_weight
    for l in range(L):
        lw = w["layers"][l]
        rows = np.flatnonzero(mask & (depth > l))
        active.append(int(rows.size))
        K = np.zeros((n, kvw))
        V = np.zeros((n, kvw))
        for (start, _), c in zip(lay["segment_slots"], caches):
            if c is not None:
                ns = c[0][l].shape[0]
                K[start : start + ns] = c[0][l][:, kc] if c[0][l].shape[1] != kvw else c[0][l]
                V[start : start + ns] = c[1][l][:, kc] if c[1][l].shape[1] != kvw else c[1][l]
        if rows.size:
            x = hidden[rows]
            xn = rmsnorm(x, cfg.rms_eps, lw["attn_norm"] if nw else None)
            K[rows] = xn @ lw["wk"][:, kc]
            V[rows] = xn @ lw["wv"][:, kc]
            if sample_rows is not None and l == L - 1:
                keep = np.isin(rows, np.asarray(sample_rows, dtype=np.int64))
                rows, x, xn = rows[keep], x[keep], xn[keep]
            q = xn @ lw["wq"][:, qc]
            qr = rope(q, pos[rows], cfg.rpe_base, dh).reshape(rows.size, H, dh)
            kr = rope(K, key_pos, cfg.rpe_base, dh).reshape(n, Hkv, dh)
            vv = V.reshape(n, Hkv, dh)
            # GQA: query head h reads kv head h // group (contiguous grouping)
            kr_h = np.repeat(kr.transpose(1, 0, 2), group, axis=0)  # [H, n, dh]
            vv_h = np.repeat(vv.transpose(1, 0, 2), group, axis=0)
            s = np.matmul(qr.transpose(1, 0, 2), kr_h.transpose(0, 2, 1)) / np.sqrt(dh)  # [H, q, n]
            ok = (pos[None, :] <= pos[rows][:, None]) & ~pad[None, :]
            s[:, ~ok] = -np.inf
            s -= s.max(axis=2, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=2, keepdims=True)
            ctx = np.matmul(p, vv_h).transpose(1, 0, 2).reshape(rows.size, H * dh)
            hidden[rows] = x + reduce(ctx @ lw["wo"][qc, :])
            x2 = hidden[rows]
            xn2 = rmsnorm(x2, cfg.rms_eps, lw["mlp_norm"] if nw else None)
            if cfg.mlp == "swiglu":
                ff = silu(xn2 @ lw["w_gate"][:, fc]) * (xn2 @ lw["w_up"][:, fc])
            else:
                ff = gelu_tanh(xn2 @ lw["w_up"][:, fc])
            hidden[rows] = x2 + reduce(ff @ lw["w_down"][fc, :])
            attn_w.append(p if keep_weights else None)
        else:
            attn_w.append(np.zeros((H, 0, n)) if keep_weights else None)
        attn_rows.append(rows)
        keys_out.append(K)
        vals_out.append(V)
    return {
        "hidden": hidden,
        "keys": keys_out,
        "values": vals_out,
        "attn": attn_w,
        "attn_rows": attn_rows,
        "active_per_layer": active,
        "computed": mask & (depth >= cfg.n_layers),
        "positions": pos.copy(),
        "question_span": lay["question_span"],
        "segment_slots": lay["segment_slots"],
    }


def logits(w: dict, cfg: OracleConfig, rows) -> np.ndarray:
    """Model.logits (model.py:94-95): rmsnorm(h) @ unembed."""
    r = np.atleast_2d(np.asarray(rows, dtype=np.float64))
    return rmsnorm(r, cfg.rms_eps, w["final_norm"] if cfg.norm_weight else None) @ w["unembed"]


def greedy_token(w: dict, cfg: OracleConfig, result: dict) -> int:
    """First decode token (model.py:455) from the question's last row."""
    q1 = result["question_span"][1]
    return int(np.argmax(logits(w, cfg, result["hidden"][q1 - 1])[0]))


def decode(w: dict, cfg: OracleConfig, keys, values, positions, valid, last_hidden, max_steps: int):
    """Greedy decode (model.py:445-484): token = argmax(logits(hidden_row));
    embed it; per layer the new row's q/k/v from the normed state, ALL keys
    (stored position-free, pads at position 0, :466) rotated at their
    positions, q at next_pos, pads masked, residual MLP; the new K/V row is
    appended (:481 append_token).  Returns (tokens, keys, values) with the
    per-layer K/V extended by max_steps rows."""
    H, Hkv, dh, d = cfg.n_heads, cfg.hkv, cfg.dh, cfg.d_model
    group = H // Hkv
    nw = cfg.norm_weight
    keys = [np.asarray(k, dtype=np.float64) for k in keys]
    values = [np.asarray(v, dtype=np.float64) for v in values]
    positions = np.asarray(positions, dtype=np.int64)
    valid = np.asarray(valid, dtype=bool)
    out = []
    if max_steps <= 0:
        return out, keys, values
    hidden_row = np.asarray(last_hidden, dtype=np.float64).reshape(1, d)
    next_pos = int(positions[valid].max()) + 1
    for _ in range(max_steps):
        token = int(np.argmax(logits(w, cfg, hidden_row)[0]))
        out.append(token)
        x = w["embed"][token][None, :]
        new_rows = []
        for l in range(cfg.n_layers):
            lw = w["layers"][l]
            xn = rmsnorm(x, cfg.rms_eps, lw["attn_norm"] if nw else None)
            q = xn @ lw["wq"]
            k_new = xn @ lw["wk"]
            v_new = xn @ lw["wv"]
            K = np.vstack([keys[l], k_new])
            V = np.vstack([values[l], v_new])
            key_pos = np.append(np.where(valid, positions, 0), next_pos)
            kr = rope(K, key_pos, cfg.rpe_base, dh).reshape(-1, Hkv, dh)
            qr = rope(q, [next_pos], cfg.rpe_base, dh).reshape(H, dh)
            kr_h = np.repeat(kr.transpose(1, 0, 2), group, axis=0)  # [H, n, dh]
            vv_h = np.repeat(V.reshape(-1, Hkv, dh).transpose(1, 0, 2), group, axis=0)
            sc = np.einsum("hd,hkd->hk", qr, kr_h) / np.sqrt(dh)
            ok = np.append(valid, True)
            sc[:, ~ok] = -np.inf
            sc -= sc.max(axis=1, keepdims=True)
            p = np.exp(sc)
            p /= p.sum(axis=1, keepdims=True)
            ctx = np.einsum("hk,hkd->hd", p, vv_h).reshape(1, H * dh)
            x = x + ctx @ lw["wo"]
            xn2 = rmsnorm(x, cfg.rms_eps, lw["mlp_norm"] if nw else None)
            if cfg.mlp == "swiglu":
                ff = silu(xn2 @ lw["w_gate"]) * (xn2 @ lw["w_up"])
            else:
                ff = gelu_tanh(xn2 @ lw["w_up"])
            x = x + ff @ lw["w_down"]
            new_rows.append((k_new, v_new))
        for l, (k_row, v_row) in enumerate(new_rows):
            keys[l] = np.vstack([keys[l], k_row])
            values[l] = np.vstack([values[l], v_row])
        positions = np.append(positions, next_pos)
        valid = np.append(valid, True)
        next_pos += 1
        hidden_row = x
    return out, keys, values


# --------------------------------------------------------------------------
# selection and scoring  (planner.py:17-34, scoring.py:45-111)
# --------------------------------------------------------------------------


def recompute_count(n: int, cfo: float) -> int:
    """planner.py:30."""
    return min(n, int(math.ceil(cfo * n - 1e-9))) if cfo > 0 else 0


def select_tokens(scores, cfo: float) -> np.ndarray:
    """planner.py:17-34: the ceil(cfo*n - 1e-9) best scores, ties to the
    lower index, returned ascending."""
    s = np.asarray(scores, dtype=np.float64)
    k = recompute_count(s.size, cfo)
    if k <= 0:
        return np.empty(0, dtype=np.int64)
    # stable sort on -score keeps equal scores in index order
    order = np.argsort(-s, kind="stable")
    return np.sort(order[:k]).astype(np.int64)


def beta(prefix_ids, prefix_weights, new_prefix) -> float:
    """scoring.py:45-56."""
    tot = sum(prefix_weights)
    if not prefix_ids or tot == 0:
        return 1.0
    keep = set(new_prefix)
    return sum(wt for cid, wt in zip(prefix_ids, prefix_weights) if cid in keep) / tot


def gamma(old_order, new_order) -> float:
    """scoring.py:59-76: discordant pairs of the common subset / C(m,2)."""
    common = set(old_order) & set(new_order)
    a = [c for c in old_order if c in common]
    rank = {c: i for i, c in enumerate(c for c in new_order if c in common)}
    m = len(a)
    if m <= 1:
        return 0.0
    disc = sum(1 for x in range(m) for y in range(x + 1, m) if rank[a[x]] > rank[a[y]])
    return disc / (m * (m - 1) / 2)


def cci(a_bar: float, b_bar: float) -> float:
    """scoring.py:85-95."""
    return 1.0 if b_bar == 0 else 1.0 / (1.0 + math.exp(-a_bar / b_bar))


def cfo(alpha: float, cci_val: float, beta_prime: float) -> float:
    """scoring.py:98-103."""
    return min(1.0, max(0.0, alpha * cci_val * (1.0 - beta_prime)))


def score_variant(prefix_ids, prefix_weights, cci_val, new_prefix, alpha):
    """scoring.py:106-111 -> (beta, gamma, beta', cfo)."""
    b = beta(prefix_ids, prefix_weights, new_prefix)
    g = gamma(prefix_ids, new_prefix)
    bp = b * (1.0 - g)
    return b, g, bp, cfo(alpha, cci_val, bp)


def chunk_hash(tokens) -> str:
    """store.py:22-27: blake2b-64 of the int64 little-endian token bytes."""
    return hashlib.blake2b(np.asarray(tokens, dtype="<i8").tobytes(), digest_size=8).hexdigest()


# --------------------------------------------------------------------------
# attention statistics  (stats.py:68-176, harness.py:331-354)
# --------------------------------------------------------------------------


def _head_mean_rows(result, layer, slots):
    rows = result["attn_rows"][layer]
    where = {int(s): i for i, s in enumerate(rows)}
    a = result["attn"][layer].mean(axis=0)
    return a[[where[int(s)] for s in slots]]


def segment_mass(result, layer, slots, spans):
    """Head-mean attention mass of each query slot onto each span's keys
    [len(slots), len(spans)] (the quantity every stat below sums)."""
    a = _head_mean_rows(result, layer, slots)
    return np.stack([a[:, s0:s1].sum(axis=1) for (s0, s1) in spans], axis=1)


def inter(result, spans, i, j, layer) -> float:
    """stats.py:68-75: mass from span j's queries onto span i's keys (i<j)."""
    a = _head_mean_rows(result, layer, range(*spans[j]))
    return float(a[:, spans[i][0] : spans[i][1]].sum())


def intra(result, spans, i, layer) -> float:
    """stats.py:78-84: strictly-lower-triangular mass inside span i."""
    s0, s1 = spans[i]
    a = _head_mean_rows(result, layer, range(s0, s1))[:, s0:s1]
    return float(np.tril(a, k=-1).sum())


def diagonal_mass(result, spans, i, layer) -> float:
    """stats.py:87-91."""
    s0, s1 = spans[i]
    a = _head_mean_rows(result, layer, range(s0, s1))[:, s0:s1]
    return float(np.trace(a))


def token_inter_scores(result, spans, i, n_layers=None) -> np.ndarray:
    """stats.py:94-106: per-token mass onto all earlier spans, layer-summed."""
    s0, s1 = spans[i]
    out = np.zeros(s1 - s0)
    if i == 0:
        return out
    cols = np.concatenate([np.arange(*spans[j]) for j in range(i)])
    L = len(result["attn"]) if n_layers is None else n_layers
    for l in range(L):
        a = _head_mean_rows(result, l, range(s0, s1))
        out += a[:, cols].sum(axis=1)
    return out


def question_inter_stream(result, spans) -> np.ndarray:
    """stats.py:160-176: [L, k] question->chunk mass per layer."""
    q0, q1 = result["question_span"]
    L = len(result["attn"])
    out = np.zeros((L, len(spans)))
    if q1 == q0:
        return out
    for l in range(L):
        present = set(int(s) for s in result["attn_rows"][l])
        qs = [s for s in range(q0, q1) if s in present]
        if not qs:
            continue
        a = _head_mean_rows(result, l, qs)
        for i, (s0, s1) in enumerate(spans):
            out[l, i] = a[:, s0:s1].sum()
    return out


def fresh_chunk_stats(result, spans, chunk_ids, i):
    """harness.py:331-354: creation-time metadata of a freshly computed chunk:
    (prefix ids, prefix weights, a_bar, b_bar, token scores)."""
    L = len(result["attn"])
    li = spans[i][1] - spans[i][0]
    a_l = np.zeros(L)
    wsum = {}
    for j in range(i):
        lj = spans[j][1] - spans[j][0]
        il = np.array([inter(result, spans, j, i, l) for l in range(L)])
        a_l += il / (li * lj)
        wsum[chunk_ids[j]] = wsum.get(chunk_ids[j], 0.0) + float(il.sum())
    b_l = np.array([intra(result, spans, i, l) for l in range(L)]) / li**2
    ids = list(dict.fromkeys(chunk_ids[:i]))
    return tuple(ids), tuple(wsum[c] for c in ids), float(a_l.mean()), float(b_l.mean()), token_inter_scores(result, spans, i)
