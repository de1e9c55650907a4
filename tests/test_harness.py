"""The bench harness against the reference's own lazymat.bench
(tests/golden/harness.json, made by tests/golden/make_golden_harness.py):
report rendering (CPU), argument validation and expression builders (CPU),
and the flop / allocation columns of run_bench for the ten canonical
expressions (GPU)."""

import json

import numpy as np
import pytest

import paper_2502_03000_b200 as lm
from conftest import GOLDEN
from paper_2502_03000_b200.harness import BenchRecord, build_expression, report, run_bench

GOLD = json.loads((GOLDEN / "harness.json").read_text())


def _records():
    return [BenchRecord(expr_id=e, size=s, mode=m, mean_seconds=t, flops=f, allocations=a, runs=r)
            for e, s, m, t, f, a, r in GOLD["synthetic"]]


def test_csv_report_matches_reference():
    assert report(_records(), format="csv") == GOLD["csv"]


def test_markdown_report_matches_reference():
    assert report(_records(), format="markdown") == GOLD["markdown"]


def test_report_rejects_unknown_format():
    with pytest.raises(ValueError):
        report(_records(), format="html")


def test_run_bench_validates_arguments():
    with pytest.raises(ValueError):
        run_bench([1], [8], runs=0, seed=42)
    with pytest.raises(ValueError):
        run_bench([1], [8], runs=1, seed=42, mode="fast")


def test_build_expression_rejects_bad_input():
    with pytest.raises(ValueError):
        build_expression(1, 3, 42)
    with pytest.raises(ValueError):
        build_expression(11, 8, 42)


@pytest.mark.parametrize("expr_id", range(1, 11))
def test_build_expression_shapes_and_determinism(expr_id):
    t1, ops1 = build_expression(expr_id, 8, 42)
    t2, ops2 = build_expression(expr_id, 8, 42)
    assert lm.infer_shape(t1) == lm.infer_shape(t2)
    for k in ops1:
        assert np.array_equal(ops1[k].to_numpy(), ops2[k].to_numpy())


@pytest.mark.gpu
def test_run_bench_counters_match_reference():
    """Flops and allocations of both arms, every canonical expression, as
    the reference's own run_bench records them."""
    recs = run_bench(list(range(1, 11)), [8, 16], runs=1, seed=42, mode="both")
    got = [[r.expr_id, r.size, r.mode, r.flops, r.allocations] for r in recs]
    assert got == GOLD["counters"]
