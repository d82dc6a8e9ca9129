"""TEST INFRASTRUCTURE: hands a device model's weights / caches to the CPU
oracle (``cachecraft_oracle``).  Used only by ``tests/`` and by
``bench.py``'s CPU-baseline leg, so the oracle runs on the SAME weights and
chunk caches as the GPU path.  Never imported by the product package."""

from __future__ import annotations

import numpy as np


def oracle_config(model, n_layers=None):
    from .cachecraft_oracle import OracleConfig

    c = model.kcfg
    return OracleConfig(n_layers=c.n_layers if n_layers is None else n_layers, n_heads=c.n_heads,
                        d_model=c.d_model, d_head=c.head_dim(), vocab_size=c.vocab_size, rpe_base=c.rpe_base,
                        n_kv_heads=c.kv_heads(), d_ff=c.ff_dim(), mlp=c.mlp, norm_weight=c.norm_weight,
                        rms_eps=c.rms_eps)


def weights_from_model(model, token_ids, n_layers=None):
    """The device model's weights as the oracle's float64 [in, out] dict
    (bf16 weights exactly as rounded on the device), with a compact embedding
    table of only the rows ``token_ids`` uses.  Returns (weights, remap):
    ``remap(tokens)`` maps real token ids to rows of the compact table.
    Uses the rank-local shape (model.kcfg), so a tensor-parallel rank
    exports its own slices; ``n_layers`` limits the export to the first
    layers."""
    import torch

    cfg = model.kcfg
    q, kv, ff, d = cfg.q_width(), cfg.kv_width(), cfg.ff_dim(), cfg.d_model

    def h(t):
        return t.double().cpu().numpy()

    layers = []
    for lw in model.w["layers"][: n_layers if n_layers is not None else len(model.w["layers"])]:
        qkv = h(lw["w_qkv"]).T
        out = {"wq": qkv[:, :q], "wk": qkv[:, q:q + kv], "wv": qkv[:, q + kv:], "wo": h(lw["w_o"]).T,
               "w_down": h(lw["w_down"]).T}
        if cfg.mlp == "swiglu":
            gu = h(lw["w_gu"]).reshape(ff // 64, 2, 64, d)
            out["w_gate"] = np.ascontiguousarray(gu[:, 0].reshape(ff, d).T)
            out["w_up"] = np.ascontiguousarray(gu[:, 1].reshape(ff, d).T)
        else:
            out["w_up"] = h(lw["w_up"]).T
        out["attn_norm"] = h(lw["attn_norm"]) if "attn_norm" in lw else np.ones(d)
        out["mlp_norm"] = h(lw["mlp_norm"]) if "mlp_norm" in lw else np.ones(d)
        layers.append(out)
    uniq = np.unique(np.concatenate([np.asarray(t, dtype=np.int64).reshape(-1) for t in token_ids]))
    idx = torch.from_numpy(uniq).to(model.w["embed"].device)
    w = {"embed": h(model.w["embed"][idx]), "layers": layers,
         "final_norm": h(model.w["final_norm"]) if "final_norm" in model.w else np.ones(d)}

    def remap(tokens):
        return np.searchsorted(uniq, np.asarray(tokens, dtype=np.int64))

    return w, remap


def cache_layers(cache, n_layers):
    """(keys, values) of a chunk cache's first ``n_layers`` layers as float64
    host arrays [n_slots, kv_width], read straight from its device payload."""
    p = cache._payload
    if p is None or not hasattr(p, "layer_rows"):
        return [np.asarray(k) for k in cache.keys[:n_layers]], [np.asarray(v) for v in cache.values[:n_layers]]
    keys = [p.layer_rows(l, 0).double().cpu().numpy() for l in range(n_layers)]
    vals = [p.layer_rows(l, 1).double().cpu().numpy() for l in range(n_layers)]
    return keys, vals


def logits_from_model(model, hidden_row, block=16384):
    """Model.logits (model.py:94-95) in float64 on the host against the
    device's unembedding (streamed to the host in vocab blocks)."""
    from .cachecraft_oracle import rmsnorm

    cfg = model.config
    fn = model.w["final_norm"].double().cpu().numpy() if "final_norm" in model.w else None
    xn = rmsnorm(np.asarray(hidden_row, dtype=np.float64).reshape(1, -1), cfg.rms_eps,
                 fn if cfg.norm_weight else None)[0]
    un = model.w["unembed_t"]  # [vocab, d]
    out = np.empty(un.shape[0])
    for i in range(0, un.shape[0], block):
        out[i:i + block] = un[i:i + block].double().cpu().numpy() @ xn
    return out
