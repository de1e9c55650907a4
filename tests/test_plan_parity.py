"""Plan parity with the reference: rule logs, kernel sequences, params,
slot shapes and describe() of every golden case (tests/golden/cases.py),
against plans the REFERENCE produced (tests/golden/plans.json).

Planning needs no device, so this runs on CPU for every case whose
rewrite does not run the structure scan; the scan cases (R9/R10 on leaf
coefficients) are covered on the GPU in tests/test_gpu_parity.py.
"""

import json
import re

import pytest

import paper_2502_03000_b200 as lm
from cases import CASES, NEEDS_SCAN
from conftest import GOLDEN

GOLD = json.loads((GOLDEN / "plans.json").read_text())

_ID_RE = re.compile(r"\bm(\d+)\b")


def normalise_ids(text: str) -> str:
    seen = {}

    def sub(m):
        seen.setdefault(m.group(1), len(seen) + 1)
        return f"m#{seen[m.group(1)]}"

    return _ID_RE.sub(sub, text)


def plan_record(plan):
    return {
        "rule_log": list(plan.rule_log),
        "kernels": [s.kernel for s in plan.steps],
        "params": [repr(tuple(s.params)) for s in plan.steps],
        "dests": [list(plan.slot_shapes[s.dest]) for s in plan.steps],
        "slot_shapes": [list(s) for s in plan.slot_shapes],
        "result_slot": plan.result_slot,
        "scalar": bool(plan.scalar_result),
        "describe": normalise_ids(plan.describe()),
    }


def test_every_case_has_a_golden():
    assert set(CASES) == set(GOLD)
    assert {k for k, v in GOLD.items() if v["needs_scan"]} == NEEDS_SCAN


@pytest.mark.parametrize("name", sorted(n for n in CASES if n not in NEEDS_SCAN))
def test_plan_matches_reference(name):
    plan = lm.rewrite(CASES[name](lm))
    got = plan_record(plan)
    want = {k: GOLD[name][k] for k in got}
    assert got == want


@pytest.mark.parametrize("name", sorted(n for n in CASES if n not in NEEDS_SCAN))
def test_rule_events_match_reference(name):
    """Planning emits one rule event per rule-log entry, in order, and
    they open the reference's own rule-event stream (run-time R10
    dispatch events follow during execution)."""
    tr = lm.with_trace(lambda: lm.rewrite(CASES[name](lm)))
    rules = [e.name for e in tr.events if e.kind == "rule"]
    gold = [ln.split("rule: ", 1)[1].split(" [")[0] for ln in GOLD[name]["trace"].splitlines() if ": rule: " in ln]
    assert rules == GOLD[name]["rule_log"]
    assert gold[: len(rules)] == rules
