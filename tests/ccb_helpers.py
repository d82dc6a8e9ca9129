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
