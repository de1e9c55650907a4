"""Pin the CPU oracle bit-for-bit against the reference's own outputs.

tests/golden/kernels.{json,npz} were produced by running the reference
``lazymat._loops`` functions (tests/golden/make_golden.py).  The C
restatement in oracle/lm_oracle.c must reproduce every output exactly
(bitwise, including pivots and return codes) before any GPU result is
compared against it.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import lm_oracle as O

MANIFEST = json.loads((GOLDEN / "kernels.json").read_text())
ARR = np.load(GOLDEN / "kernels.npz")


def _by_kind(kind):
    return [r for r in MANIFEST if r["kind"] == kind]


def _a(rec, key):
    return ARR[rec[key]]


def _bits_equal(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.int64), y.view(np.int64))


def test_manifest_covers_every_loop_family():
    kinds = {r["kind"] for r in MANIFEST}
    assert kinds == {"analyze", "fused", "gemm", "gemv", "syrk", "diag_scale", "dotprod",
                     "triple", "lu", "band", "tri", "copyops"}


@pytest.mark.parametrize("rec", _by_kind("analyze"), ids=lambda r: r["name"])
def test_analyze(rec):
    assert O.analyze(_a(rec, "a"), rec["square"]) == (rec["lbw"], rec["ubw"], rec["sym"])


@pytest.mark.parametrize("rec", _by_kind("fused"), ids=lambda r: r["name"])
def test_fused(rec):
    srcs = [_a(rec, f"s{k}") for k in range(rec["nterm"])]
    if rec["name"] == "fused/6":
        srcs[1] = np.ascontiguousarray(srcs[1].T).T  # same values, C-order .T view
    out = np.zeros_like(_a(rec, "out"), order="F")
    O.fused(rec["coeffs"], srcs, out)
    assert _bits_equal(out, _a(rec, "out"))


@pytest.mark.parametrize("rec", _by_kind("gemm"), ids=lambda r: r["name"])
def test_gemm(rec):
    a, b = _a(rec, "a"), _a(rec, "b")
    out = np.zeros_like(_a(rec, "out"), order="F")
    O.gemm(np.ascontiguousarray(a.T).T, b, out)  # strided operand read in place
    assert _bits_equal(out, _a(rec, "out"))


@pytest.mark.parametrize("rec", _by_kind("gemv"), ids=lambda r: r["name"])
def test_gemv(rec):
    out = np.zeros_like(_a(rec, "out"))
    O.gemv(_a(rec, "a"), _a(rec, "x"), out, rec["trans"])
    assert _bits_equal(out, _a(rec, "out"))


@pytest.mark.parametrize("rec", _by_kind("syrk"), ids=lambda r: r["name"])
def test_syrk(rec):
    out = np.zeros_like(_a(rec, "out"), order="F")
    O.syrk(_a(rec, "a"), out)
    assert _bits_equal(out, _a(rec, "out"))
    assert _bits_equal(out, out.T)


@pytest.mark.parametrize("rec", _by_kind("diag_scale"), ids=lambda r: r["name"])
def test_diag_scale(rec):
    out = np.zeros_like(_a(rec, "out"), order="F")
    O.diag_scale(_a(rec, "d"), _a(rec, "b"), rec["side"], out)
    assert _bits_equal(out, _a(rec, "out"))


@pytest.mark.parametrize("rec", _by_kind("dotprod"), ids=lambda r: r["name"])
def test_diag_and_trace_of_product(rec):
    a, b = _a(rec, "a"), _a(rec, "b")
    d = np.zeros_like(_a(rec, "diag"))
    O.diag_of_product(a, b, d)
    assert _bits_equal(d, _a(rec, "diag"))
    t = O.trace_of_product(a, b)
    assert _bits_equal(t, rec["trace"])


@pytest.mark.parametrize("rec", _by_kind("triple"), ids=lambda r: r["name"])
def test_triple(rec):
    assert _bits_equal(O.triple_diag_dot(_a(rec, "a"), _a(rec, "d"), _a(rec, "c")), rec["out"])


@pytest.mark.parametrize("rec", _by_kind("lu"), ids=lambda r: r["name"])
def test_lu_factor_and_solve(rec):
    rc, lu, piv = O.lu_factor(_a(rec, "a"))
    assert rc == rec["rc"]
    upto = rc if rc else len(piv)  # on failure, pivots of columns 0..rc-1 were written
    assert np.array_equal(piv[:upto], _a(rec, "piv")[:upto])
    if rc == 0:
        assert _bits_equal(lu, _a(rec, "lu"))
        x = np.array(_a(rec, "b"), order="F")
        O.lu_solve(lu, piv, x)
        assert _bits_equal(x, _a(rec, "x"))


def test_lu_golden_includes_singular_and_pivoting():
    recs = _by_kind("lu")
    assert any(r["rc"] for r in recs)
    assert any(not np.array_equal(ARR[r["piv"]], np.arange(len(ARR[r["piv"]])))
               for r in recs if r["rc"] == 0)


@pytest.mark.parametrize("rec", _by_kind("band"), ids=lambda r: r["name"])
def test_band(rec):
    x = np.array(_a(rec, "b"), order="F")
    rc = O.band_solve(_a(rec, "a"), x, rec["kl"], rec["ku"])
    assert rc == rec["rc"]
    if rc == 0:
        assert _bits_equal(x, _a(rec, "x"))


@pytest.mark.parametrize("rec", _by_kind("tri"), ids=lambda r: r["name"])
def test_tri(rec):
    x = np.array(_a(rec, "b"), order="F")
    rc = O.tri_solve(_a(rec, "a"), x, rec["upper"])
    assert rc == rec["rc"]
    if rc == 0:
        assert _bits_equal(x, _a(rec, "x"))


@pytest.mark.parametrize("rec", _by_kind("copyops"), ids=lambda r: r["name"])
def test_copy_ops(rec):
    a = _a(rec, "a")
    t = np.zeros((a.shape[1], a.shape[0]), order="F")
    O.transpose_copy(a, t)
    assert _bits_equal(t, _a(rec, "t"))
    d = _a(rec, "d")
    dm = np.ones((d.shape[0], d.shape[0]), order="F")
    O.diag_materialise(d, dm)
    assert _bits_equal(dm, _a(rec, "dm"))


def test_program_matches_axpby_family():
    """The extension program interpreter, restricted to a linear
    combination, reproduces the reference fused loops bitwise."""
    rec = _by_kind("fused")[3]
    srcs = [_a(rec, f"s{k}") for k in range(rec["nterm"])]
    ops, args, consts = [], [], []
    for k, c in enumerate(rec["coeffs"]):
        consts.append(c)
        ops += [1, 0, 4]
        args += [len(consts) - 1, k, 0]
        if k:
            ops.append(2)
            args.append(0)
    out = np.zeros_like(_a(rec, "out"), order="F")
    O.program(ops, args, consts, srcs, out)
    assert _bits_equal(out, _a(rec, "out"))
