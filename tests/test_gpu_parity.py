"""GPU parity: every golden case evaluated on the B200 through the C ABI.

For each case of tests/golden/cases.py we compare with what the
REFERENCE produced (tests/golden/plans.{json,npz}):
  * the full plan (now including the R9/R10 cases whose rewrite runs the
    device structure scan);
  * the traced event stream (kernel / rule / detect / alloc / free, ids
    normalised) and the counters -- flops, allocations, kernel calls;
  * the evaluate() value: bit-exact where the reference's arithmetic is
    reproduced operation by operation (element-wise, diag scaling, all
    solves), normwise <= 1e-12 where a reduction is reassociated (GEMM,
    GEMV, SYRK, trace/diag of a product);
  * the naive arm (value within 1e-12 normwise, or the same error).
"""

import json
import re

import numpy as np
import pytest

import paper_2502_03000_b200 as lm
from cases import CASES
from conftest import GOLDEN
from test_plan_parity import plan_record

pytestmark = pytest.mark.gpu

GOLD = json.loads((GOLDEN / "plans.json").read_text())
ARR = np.load(GOLDEN / "plans.npz")

_REASSOC = {"gemm", "syrk", "trace_of_product", "diag_of_product", "triple_diag_dot"}
_EV_ID_RE = re.compile(r"id=(\d+)")


def normalise_trace(text: str) -> str:
    seen = {}

    def sub(m):
        seen.setdefault(m.group(1), len(seen) + 1)
        return f"id=#{seen[m.group(1)]}"

    return _EV_ID_RE.sub(sub, text)


def _host(res):
    if isinstance(res, float):
        return np.array([[res]])
    return res.to_numpy()


def _close(got, want, exact: bool, tol=1e-12):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    if exact:
        assert np.array_equal(got.view(np.int64), want.view(np.int64)), \
            f"not bit-identical: max|d|={np.max(np.abs(got - want)) if got.size else 0}"
    else:
        scale = max(float(np.max(np.abs(want))) if want.size else 0.0, 1e-300)
        gap = float(np.max(np.abs(got - want))) / scale if want.size else 0.0
        assert gap <= tol, f"normwise gap {gap:.3e} > {tol}"


@pytest.mark.parametrize("name", sorted(CASES))
def test_case_matches_reference(name):
    gold = GOLD[name]
    tree = CASES[name](lm)
    plan = lm.rewrite(tree)
    rec = plan_record(plan)
    assert rec == {k: gold[k] for k in rec}
    tr = lm.with_trace(lambda: lm.evaluate(tree))
    assert normalise_trace(lm.render_trace(tr.events)) == gold["trace"]
    assert [tr.counters.flops, tr.counters.allocations, tr.counters.kernel_calls] == gold["counters"]
    want = np.array([[gold["value"]]]) if "value" in gold else ARR[f"{name}/evaluate"]
    exact = not (set(gold["kernels"]) & _REASSOC)
    _close(_host(tr.result), want, exact)


@pytest.mark.parametrize("name", sorted(CASES))
def test_naive_arm_matches_reference(name):
    gold = GOLD[name]
    tree = CASES[name](lm)
    if "naive_error" in gold:
        with pytest.raises(getattr(lm, gold["naive_error"])):
            lm.naive_evaluate(tree)
        return
    tr = lm.with_trace(lambda: lm.naive_evaluate(tree))
    assert normalise_trace(lm.render_trace(tr.events)) == gold["naive_trace"]
    assert [tr.counters.flops, tr.counters.allocations, tr.counters.kernel_calls] == gold["naive_counters"]
    want = np.array([[gold["naive_value"]]]) if "naive_value" in gold else ARR[f"{name}/naive"]
    _close(_host(tr.result), want, exact=False, tol=1e-10 if "inverse" in gold["naive_trace"] else 1e-12)
