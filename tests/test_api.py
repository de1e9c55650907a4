"""Matrix and trace API behaviours against the reference's own outputs
(tests/golden/api.json, made by tests/golden/make_golden_api.py):
fills, column-major values, debug_format, storage identity, trace
rendering and counters, exact structure analysis."""

import json
import re

import numpy as np
import pytest
import torch

import paper_2502_03000_b200 as lm
from conftest import GOLDEN
from paper_2502_03000_b200.errors import DimensionError, LengthError
from paper_2502_03000_b200.trace import TraceEvent, current_collector, render_trace, with_trace

GOLD = json.loads((GOLDEN / "api.json").read_text())
_ID = re.compile(r"id=(\d+)")


def _norm(text):
    seen = {}
    return _ID.sub(lambda m: "id=#%d" % seen.setdefault(m.group(1), len(seen) + 1), text)


@pytest.mark.parametrize("name", sorted(GOLD["traces"]))
def test_render_trace_of_reference_events(name):
    g = GOLD["traces"][name]
    events = [TraceEvent(seq, kind, nm, detail) for seq, kind, nm, detail in g["events"]]
    assert render_trace(events) == g["rendered"]


def test_render_empty_trace_is_empty():
    assert render_trace([]) == ""


def test_values_fill_is_column_major():
    g = GOLD["values_2x3"]
    m = lm.make_matrix(2, 3, fill="values", values=[1.0, 2.5, -3.0, 4.0, 0.125, 6.0])
    assert m.to_values() == g["to_values"]
    assert m.debug_format() == g["debug_format"]
    assert [[m.element(i, j) for j in range(3)] for i in range(2)] == g["elements"]


def test_values_length_mismatch():
    with pytest.raises(LengthError):
        lm.make_matrix(2, 2, fill="values", values=[1.0, 2.0, 3.0])


def test_random_fill_is_the_references_stream_and_needs_a_seed():
    assert lm.make_matrix(3, 2, fill="random", seed=11).to_values() == GOLD["random_3x2_seed11"]
    with pytest.raises(ValueError):
        lm.make_matrix(3, 2, fill="random")


def test_identity_fill_requires_square():
    assert lm.make_matrix(3, 3, fill="identity").to_values() == GOLD["identity_3"]
    with pytest.raises(DimensionError):
        lm.make_matrix(2, 3, fill="identity")


def test_storage_is_fortran_float64_and_ids_name_storage():
    a = lm.make_matrix(4, 3, fill="random", seed=1)
    b = lm.make_matrix(4, 3, fill="random", seed=1)
    assert a.data.dtype == torch.float64 and a.data.stride() == (1, 4)
    assert a.to_values() == b.to_values() and a.id != b.id
    c = a.copy()
    assert c.id != a.id and c.to_values() == a.to_values()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD["traces"]))
def test_traced_evaluation_matches_reference(name):
    a = lm.make_matrix(6, 6, fill="random", seed=3)
    b = lm.make_matrix(6, 6, fill="random", seed=4)
    v = lm.make_matrix(6, 1, fill="random", seed=5)
    expr = {"weighted_sum": lm.add(lm.smul(0.25, a), lm.smul(0.75, b)),
            "chain": lm.matmul(lm.matmul(a, b), v),
            "trace_product": lm.trace(lm.matmul(a, b))}[name]
    t = with_trace(lambda: lm.evaluate(expr))
    g = GOLD["traces"][name]
    assert _norm(render_trace(t.events)) == _norm(g["rendered"])
    assert [t.counters.flops, t.counters.allocations, t.counters.kernel_calls] == g["counters"]
    # tracing changes no bits
    plain = lm.evaluate(expr)
    if isinstance(plain, float):
        assert plain == t.result
    else:
        assert torch.equal(plain.data, t.result.data)


@pytest.mark.gpu
def test_default_collector_is_inert():
    a = lm.make_matrix(5, 5, fill="random", seed=2)
    lm.evaluate(a * a)
    assert not current_collector().active


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD["structure"]))
def test_analyze_structure_matches_reference(name):
    g = GOLD["structure"][name]
    info = lm.analyze_structure(lm.DenseMatrix(np.asfortranarray(np.array(g["matrix"]))))
    assert [info.is_square, info.lower_bandwidth, info.upper_bandwidth, info.is_upper_triangular,
            info.is_lower_triangular, info.is_symmetric] == g["info"]
