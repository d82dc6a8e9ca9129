"""Shared test helpers (no reference imports: the GPU box has no /root/reference)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_path(name):
    return os.path.join(GOLDEN, name)


def load_json(name):
    with open(golden_path(name)) as fh:
        return json.load(fh)


def oracle_weights(model, token_ids):
    """The device model's weights as the oracle's float64 [in, out] dict
    (bf16 weights exactly as rounded on the device), with a compact embedding
    table of only the rows ``token_ids`` uses.  Returns (weights, remap):
    ``remap(tokens)`` maps real token ids to rows of the compact table.
    Uses the rank-local shape (model.kcfg) so a tensor-parallel rank exports
    its own slices."""
    import numpy as np
    import torch

    cfg = model.kcfg
    q, kv, ff, d = cfg.q_width(), cfg.kv_width(), cfg.ff_dim(), cfg.d_model

    def h(t):
        return t.double().cpu().numpy()

    layers = []
    for lw in model.w["layers"]:
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


def oracle_config(model, n_layers=None):
    from oracle import cachecraft_oracle as O

    c = model.kcfg
    return O.OracleConfig(n_layers=c.n_layers if n_layers is None else n_layers, n_heads=c.n_heads,
                          d_model=c.d_model, d_head=c.head_dim(), vocab_size=c.vocab_size, rpe_base=c.rpe_base,
                          n_kv_heads=c.kv_heads(), d_ff=c.ff_dim(), mlp=c.mlp, norm_weight=c.norm_weight,
                          rms_eps=c.rms_eps)


def oracle_logits(model, hidden_row, block=16384):
    """Model.logits (model.py:94-95) in float64 on the host against the
    device's unembedding (streamed to the host in vocab blocks)."""
    import numpy as np

    from oracle import cachecraft_oracle as O

    cfg = model.config
    fn = model.w["final_norm"].double().cpu().numpy() if "final_norm" in model.w else None
    xn = O.rmsnorm(np.asarray(hidden_row, dtype=np.float64).reshape(1, -1), cfg.rms_eps,
                   fn if cfg.norm_weight else None)[0]
    un = model.w["unembed_t"]  # [vocab, d]
    out = np.empty(un.shape[0])
    for i in range(0, un.shape[0], block):
        out[i:i + block] = un[i:i + block].double().cpu().numpy() @ xn
    return out


def rel_err(a, b):
    import numpy as np

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def row_rel_err(a, b):
    """Worst per-row relative error (rows with a zero reference are skipped)."""
    import numpy as np

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b, axis=1)
    ok = den > 0
    if not ok.any():
        return 0.0
    return float((np.linalg.norm(a - b, axis=1)[ok] / den[ok]).max())


def record_measurement(name, payload):
    """Append a measured parity figure to $CCB_PARITY_OUT (a JSON-lines file)
    when set, so the GPU run leaves its numbers behind for profiles/."""
    import json

    path = os.environ.get("CCB_PARITY_OUT")
    if not path:
        return
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "a") as fh:
        fh.write(json.dumps({"test": name, **payload}) + "\n")
