"""Trace synthesis (host logic) against the reference's own generator."""
import numpy as np

from ccb_helpers import load_json
from paper_2502_15734_b200 import harness


def test_gen_synthetic_reproduces_reference_trace():
    g = load_json("replay.json")
    tr = harness.gen_synthetic(12, 1.2, 3, 14, chunk_len_range=(16, 40), seed=3, question_len_range=(4, 8))
    assert [r.chunk_ids for r in tr.records] == [r["chunks"] for r in g["trace"]]
    assert [r.question.tolist() for r in tr.records] == [r["q"] for r in g["trace"]]
    assert [r.arrival_s for r in tr.records] == [r["arrival"] for r in g["trace"]]
    assert {str(k): v.tolist() for k, v in tr.corpus.items()} == g["corpus"]
    assert harness.top_share(tr) == g["top_share"]


def test_fit_zipf_skew_matches_reference():
    g = load_json("replay.json")
    assert harness.fit_zipf_skew(60, 5, 40, target_share=0.6, seed=3, iterations=10) == g["skew"]
