"""400 seeded random expression trees (tests/golden/fuzz_trees.py): the
rendering, validate() shape or error (type, message, error path) and
infer_shape equal the REFERENCE's, tree by tree
(tests/golden/fuzz_trees.json, made by make_golden_fuzz.py)."""

import json

import numpy as np
import pytest

import paper_2502_03000_b200 as lm
from conftest import GOLDEN
from fuzz_trees import record, trees, value_record

GOLD = json.loads((GOLDEN / "fuzz_trees.json").read_text())


def test_random_trees_match_reference():
    got = record(lm)
    want = GOLD["trees"]
    assert len(got) == len(want)
    bad = [(i, g, w) for i, (g, w) in enumerate(zip(got, want)) if g != w]
    assert not bad, bad[:3]


@pytest.mark.gpu
def test_random_trees_evaluate_like_reference():
    """Every valid tree evaluates to the reference's value (normwise <= 1e-12:
    GEMM-family reductions may reassociate) or raises the same error."""
    bad = []
    for i, (t, want) in enumerate(zip(trees(lm), GOLD["values"])):
        if want is None:
            continue
        got = value_record(lm, t)
        if got[0] != want[0] or (got[0] == "error" and got[1] != want[1]):
            bad.append((i, got, want))
            continue
        if got[0] == "ok":
            g, w = np.array(got[1]), np.array(want[1])
            scale = max(float(np.max(np.abs(w))), 1e-300)
            if g.shape != w.shape or float(np.max(np.abs(g - w))) > 1e-12 * scale:
                bad.append((i, "value", float(np.max(np.abs(g - w))) / scale))
    assert not bad, bad[:3]
