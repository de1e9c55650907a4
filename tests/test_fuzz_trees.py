"""400 seeded random expression trees (tests/golden/fuzz_trees.py): the
rendering, validate() shape or error (type, message, error path) and
infer_shape equal the REFERENCE's, tree by tree
(tests/golden/fuzz_trees.json, made by make_golden_fuzz.py)."""

import json

import paper_2502_03000_b200 as lm
from conftest import GOLDEN
from fuzz_trees import record

GOLD = json.loads((GOLDEN / "fuzz_trees.json").read_text())


def test_random_trees_match_reference():
    got = record(lm)
    assert len(got) == len(GOLD)
    bad = [(i, g, w) for i, (g, w) in enumerate(zip(got, GOLD)) if g != w]
    assert not bad, bad[:3]
