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
    from oracle.from_device import weights_from_model

    return weights_from_model(model, token_ids)


def oracle_config(model, n_layers=None):
    from oracle.from_device import oracle_config as f

    return f(model, n_layers)


def oracle_logits(model, hidden_row):
    from oracle.from_device import logits_from_model

    return logits_from_model(model, hidden_row)


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
