"""Pins of the point-adjusted evaluator oracle (NEXT-4, R-21)."""
import json
import os

import numpy as np
import pytest

from oracle import enova_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _seq(case):
    n = case["n"]
    lab = np.zeros(n, dtype=np.int8)
    for a, b in case["truth_segments"]:
        lab[a:b + 1] = 1
    pred = np.zeros(n, dtype=np.int8)
    pred[case["pred_points"]] = 1
    return lab, pred


@pytest.mark.parametrize("case", GOLD["point_adjust"], ids=lambda c: c["cite"])
def test_spec_point_adjust_examples(case):
    lab, pred = _seq(case)
    tp, fp, fn, tn = O.point_adjusted_counts(lab, pred)
    p, r, f1 = O.precision_recall_f1(tp, fp, fn)
    for k, v in (("precision", p), ("recall", r), ("f1", f1), ("tp", tp), ("fp", fp), ("fn", fn),
                 ("tn", tn)):
        if k in case:
            assert v == pytest.approx(case[k], abs=1e-12), k


def test_length_mismatch_is_an_error():
    with pytest.raises(ValueError):
        O.point_adjusted_counts([0, 1], [0])


def test_point_adjust_invariants():
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 200))
        lab = (rng.random(n) < rng.uniform(0, 0.5)).astype(np.int8)
        pred = (rng.random(n) < rng.uniform(0, 0.5)).astype(np.int8)
        tp, fp, fn, tn = O.point_adjusted_counts(lab, pred)
        assert tp + fn == int(lab.sum()) and fp + tn == n - int(lab.sum())
        # adjustment never lowers recall, never changes false positives
        raw_tp = int((lab & pred).sum())
        assert tp >= raw_tp and fp == int(((1 - lab) & pred).sum())
        # a segment is either fully counted or fully missed
        # (recompute per segment from scratch)
        i = 0
        seg_tp = seg_fn = 0
        while i < n:
            if lab[i]:
                j = i
                while j < n and lab[j]:
                    j += 1
                if pred[i:j].any():
                    seg_tp += j - i
                else:
                    seg_fn += j - i
                i = j
            else:
                i += 1
        assert (seg_tp, seg_fn) == (tp, fn)
        # predicting everything gives recall 1
        assert O.point_adjusted_counts(lab, np.ones(n, np.int8))[2] == 0
