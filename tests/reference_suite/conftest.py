"""Runs the reference's own unit tests UNMODIFIED against the drop-in.

The ``test_*.py`` files in this directory are verbatim copies of
``/root/reference/pkg/tests/`` (vendored test infrastructure, not product
code: the GPU box has no /root/reference).  This conftest makes
``import cachecraft`` / ``from cachecraft.<sub> import ...`` resolve to
``paper_2502_15734_b200`` so the reference's assertions execute on the B200
engine (fp64 mode, the reference's default ModelConfig), and provides the
fixtures the reference's conftest.py defines (toy_config, model, rng).

Every test here needs the GPU (the drop-in has no CPU path) and is marked
``gpu``.  Files listed in ``collect_ignore`` exercise reference subsystems
outside the hot path; each entry says why.
"""
import os
import sys
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2502_15734_b200 as _cc  # noqa: E402

_SUBMODULES = ("errors", "model", "planner", "rpe", "scoring", "stats", "store", "tiers", "harness")

# Reference names deliberately NOT in the drop-in (outside the hot path,
# SURVEY.md §2 out-of-scope rows).  They resolve to a stub so the test modules
# import; the tests that call them are skipped below, each with its reason.
OUT_OF_SCOPE = {
    "calibrate_alpha": "offline alpha calibration loop (scoring.py:114-152), not on the prefill path",
    "evaluate_grid": "offline alpha calibration loop (scoring.py:114-152), not on the prefill path",
    "select_alpha": "offline alpha calibration loop (scoring.py:114-152), not on the prefill path",
    "plan_to_json": "plan JSON export of the CLI (planner.py:218-264), not on the prefill path",
    "plan_from_json": "plan JSON import of the CLI (planner.py:218-264), not on the prefill path",
}
SKIPPED_TESTS = {
    # fails on the unmodified reference too (its export_report writes the
    # tokens_hit_total / tokens_hit_recomputed columns this header omits;
    # SURVEY Appendix A probe P0: 199/200); the drop-in writes the
    # reference's columns
    "test_harness.py::TestReportExport::test_empty_report_writes_header_only":
        "the reference fails this test itself (CSV header, SURVEY P0)",
    "test_scoring.py::TestCalibration": OUT_OF_SCOPE["calibrate_alpha"],
    "test_planner.py::TestPlanSerialization::test_json_round_trip_keeps_planning_fields": OUT_OF_SCOPE["plan_to_json"],
}


def _stub(name):
    def f(*a, **k):
        raise NotImplementedError(f"{name}: {OUT_OF_SCOPE[name]}")

    return f


_alias = types.ModuleType("cachecraft")
_alias.__dict__.update({k: v for k, v in vars(_cc).items() if not k.startswith("__")})
for _n in OUT_OF_SCOPE:
    if not hasattr(_cc, _n):
        setattr(_alias, _n, _stub(_n))
sys.modules.setdefault("cachecraft", _alias)
for _name in _SUBMODULES:
    sys.modules.setdefault(f"cachecraft.{_name}", getattr(__import__(f"paper_2502_15734_b200.{_name}"), _name))

collect_ignore = [
    # KVC1 model-config / raw container helpers of the CLI (cli.py); the pool
    # snapshot uses the same container format through VariantStore.snapshot
    "test_serialize.py",
    # the discrete-event tier simulator (simulate, Timeline, timeline_to_csv,
    # fallback_decision, tiers.py:74-207, :260-299): the tiers here are real
    # (engine layer-wise preload, tiers.demote_slow_hits); place_and_migrate
    # and preload_depth are pinned by tests/test_tiers_host.py fixtures
    "test_tiers.py",
]


def pytest_collection_modifyitems(config, items):
    here = os.path.dirname(os.path.abspath(__file__))
    for item in items:
        if str(item.fspath).startswith(here):
            item.add_marker(pytest.mark.gpu)
            for key, why in SKIPPED_TESTS.items():
                if key in item.nodeid:
                    item.add_marker(pytest.mark.skip(reason="out of scope: " + why))


@pytest.fixture(scope="session")
def toy_config():
    return _cc.ModelConfig()


@pytest.fixture(scope="session")
def model(toy_config):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("the drop-in runs on the GPU only")
    return _cc.build_model(toy_config)


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)
