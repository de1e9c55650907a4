"""Expression cases shared by the golden generator and the parity tests.

Every case is a function ``case(api) -> tree`` that builds its operands
and its expression tree through the public names both packages export
(the reference ``lazymat`` and ``paper_2502_03000_b200``), so the same
code yields the reference's plan/values (tests/golden/make_golden.py,
run in the build container) and ours (tests/test_plan_parity.py,
tests/test_gpu_parity.py).

Operands are seeded; host-side constructions (boosted diagonals,
tridiagonals, triangular and symmetric matrices) are computed in numpy
and handed over through ``make_matrix(..., "values", values=...)`` so
no case depends on how either package stores its buffers.

``needs_scan`` marks cases whose REWRITE already runs the structure
scan (R9/R10 on a leaf coefficient): the reference does that on the
host, we do it with a device kernel, so those plans can only be
compared where a GPU is present.
"""

from __future__ import annotations

import numpy as np


def _host(api, arr):
    arr = np.asarray(arr, dtype=np.float64)
    return api.make_matrix(arr.shape[0], arr.shape[1], "values",
                           values=list(arr.ravel(order="F")))


def _rand(seed, r, c):
    return np.random.default_rng(seed).random((r, c))


def _boosted(seed, n):
    return _rand(seed, n, n) + n * np.eye(n)


def _tridiag(seed, n):
    a = _rand(seed, n, n)
    i, j = np.indices((n, n))
    a[abs(i - j) > 1] = 0.0
    a[np.diag_indices(n)] += 2 * n
    return a


def _mat(api, r, c, seed):
    return api.make_matrix(r, c, "random", seed=seed)


CASES = {}
NEEDS_SCAN = set()


def case(name, needs_scan=False):
    def deco(fn):
        CASES[name] = fn
        if needs_scan:
            NEEDS_SCAN.add(name)
        return fn
    return deco


# ---- R1 / R2 element-wise ---------------------------------------------------

@case("r1_weighted_sum")
def _(api):
    return api.add(api.smul(0.4, _mat(api, 6, 5, 1)), api.smul(0.6, _mat(api, 6, 5, 2)))


@case("r1_nested_scalars_sub")
def _(api):
    x, y = _mat(api, 4, 4, 3), _mat(api, 4, 4, 4)
    return api.sub(api.smul(2.0, api.smul(3.0, x)), y)


@case("r1_six_terms")
def _(api):
    ms = [_mat(api, 5, 3, 10 + k) for k in range(6)]
    t = api.smul(0.5, ms[0])
    for k, c in enumerate([-1.0, 2.0, 0.25, 1.0, -0.75], start=1):
        t = api.add(t, api.smul(c, ms[k]))
    return t


@case("r1_operator_sugar")
def _(api):
    a, b, c = _mat(api, 7, 7, 5), _mat(api, 7, 7, 6), _mat(api, 7, 7, 7)
    return 0.3 * a - b + (-c) * 2.0


@case("bare_leaf_copy")
def _(api):
    return api.leaf(_mat(api, 3, 2, 1))


@case("r2_col_plus_row_t")
def _(api):
    a, b = _mat(api, 5, 5, 1), _mat(api, 5, 5, 2)
    return api.add(api.col_of(a, 1), api.transpose(api.row_of(b, 2)))


@case("r2_double_transpose")
def _(api):
    return api.transpose(api.transpose(api.col_of(_mat(api, 4, 4, 1), 0)))


@case("r2_same_view_twice")
def _(api):
    a = _mat(api, 4, 4, 1)
    return api.add(api.col_of(a, 0), api.col_of(a, 0))


@case("r2_transposed_leaf_sum")
def _(api):
    a, b = _mat(api, 6, 4, 8), _mat(api, 4, 6, 9)
    return api.add(api.transpose(a), api.smul(2.0, b))


@case("r2_view_objects")
def _(api):
    a = _mat(api, 6, 6, 21)
    return api.add(api.leaf(api.col_view(a, 2)), api.leaf(api.row_view(a, 3).transpose_view()))


@case("transpose_of_computed")
def _(api):
    a, b = _mat(api, 5, 3, 1), _mat(api, 3, 4, 2)
    return api.transpose(api.matmul(a, b))


@case("colview_of_computed")
def _(api):
    a, b = _mat(api, 5, 3, 1), _mat(api, 3, 4, 2)
    return api.col_of(api.matmul(a, b), 2)


@case("rowview_of_sum")
def _(api):
    a, b = _mat(api, 5, 4, 1), _mat(api, 5, 4, 2)
    return api.add(api.row_of(api.add(a, b), 1), api.row_of(a, 0))


# ---- R3 / R4 / R5 -----------------------------------------------------------

@case("r3_left_golden")
def _(api):
    d = api.make_matrix(2, 2, "values", values=[1, 0, 0, 2])
    b = api.make_matrix(2, 2, "values", values=[5, 7, 6, 8])
    return api.matmul(api.diagmat(d), b)


@case("r3_left_vector")
def _(api):
    return api.matmul(api.diagmat(_mat(api, 6, 1, 3)), _mat(api, 6, 5, 4))


@case("r3_right_vector")
def _(api):
    return api.matmul(_mat(api, 3, 4, 3), api.diagmat(_mat(api, 4, 1, 2)))


@case("r3_right_rowvector")
def _(api):
    return api.matmul(_mat(api, 3, 4, 3), api.diagmat(_mat(api, 1, 4, 5)))


@case("r3_diag_of_square")
def _(api):
    return api.matmul(api.diagmat(_mat(api, 5, 5, 6)), _mat(api, 5, 5, 7))


@case("r3_diag_of_computed")
def _(api):
    a, b = _mat(api, 4, 4, 1), _mat(api, 4, 4, 2)
    return api.matmul(api.diagmat(api.add(a, b)), b)


@case("r4_golden")
def _(api):
    a = api.make_matrix(2, 2, "values", values=[1, 3, 2, 4])
    b = api.make_matrix(2, 2, "values", values=[5, 7, 6, 8])
    return api.diagmat(api.matmul(a, b))


@case("r4_rect_factors")
def _(api):
    return api.diagmat(api.matmul(_mat(api, 6, 9, 1), _mat(api, 9, 6, 2)))


@case("r4_not_square_product")
def _(api):
    return api.diagmat(api.matmul(_mat(api, 4, 3, 1), _mat(api, 3, 1, 2)))


@case("r5_golden")
def _(api):
    a = api.make_matrix(2, 2, "values", values=[1, 3, 2, 4])
    b = api.make_matrix(2, 2, "values", values=[5, 7, 6, 8])
    return api.trace(api.matmul(a, b))


@case("r5_rect")
def _(api):
    return api.trace(api.matmul(_mat(api, 8, 13, 6), _mat(api, 13, 8, 7)))


@case("r5_with_transpose")
def _(api):
    a = _mat(api, 6, 6, 1)
    return api.trace(api.matmul(a, api.transpose(a)))


@case("r5_chain_reorders")
def _(api):
    a, b, c = _mat(api, 6, 6, 1), _mat(api, 6, 4, 2), _mat(api, 4, 6, 3)
    return api.trace(api.matmul(api.matmul(a, b), c))


@case("trace_plain")
def _(api):
    return api.trace(_mat(api, 7, 7, 4))


@case("trace_of_sum")
def _(api):
    return api.trace(api.add(_mat(api, 5, 5, 1), _mat(api, 5, 5, 2)))


# ---- R6 chains ----------------------------------------------------------------

def _family(api, m, base_seed=50):
    shapes = [(m, m), (m, m // 2), (m // 2, m // 3), (m // 3, m // 4)]
    return [api.make_matrix(r, c, "random", seed=base_seed + i) for i, (r, c) in enumerate(shapes)]


@case("r6_family_12")
def _(api):
    ms = _family(api, 12)
    return api.matmul(api.matmul(api.matmul(ms[0], ms[1]), ms[2]), ms[3])


@case("r6_family_24")
def _(api):
    ms = _family(api, 24, 84)
    return api.matmul(api.matmul(api.matmul(ms[0], ms[1]), ms[2]), ms[3])


@case("r6_tie_leftmost")
def _(api):
    return api.matmul(api.matmul(_mat(api, 2, 100, 1), _mat(api, 100, 100, 2)), _mat(api, 100, 2, 3))


@case("r6_abcv")
def _(api):
    a, b, c, v = (_mat(api, 16, 16, 1), _mat(api, 16, 16, 2), _mat(api, 16, 16, 3), _mat(api, 16, 1, 4))
    return api.matmul(api.matmul(api.matmul(a, b), c), v)


@case("r6_xyz")
def _(api):
    x, y, z = _mat(api, 40, 5, 1), _mat(api, 5, 40, 2), _mat(api, 40, 5, 3)
    return api.matmul(api.matmul(x, y), z)


@case("two_factor_gemm")
def _(api):
    return api.matmul(_mat(api, 3, 4, 1), _mat(api, 4, 5, 2))


@case("gemm_transposed_left")
def _(api):
    a, b = _mat(api, 9, 5, 1), _mat(api, 9, 6, 2)
    return api.matmul(api.transpose(a), b)


@case("chain_with_diag_middle")
def _(api):
    a, b, d = _mat(api, 6, 6, 1), _mat(api, 6, 6, 2), _mat(api, 6, 1, 3)
    return api.matmul(api.matmul(a, api.diagmat(d)), b)


@case("product_of_sums")
def _(api):
    a, b = _mat(api, 9, 9, 1), _mat(api, 9, 9, 2)
    return api.matmul(api.add(a, b), api.matmul(a, b))


@case("scaled_product_plus")
def _(api):
    a, b = _mat(api, 12, 12, 5), _mat(api, 12, 12, 6)
    return api.add(api.smul(0.25, api.matmul(a, b)), api.smul(3.0, a))


@case("matmul_chain_pairs")
def _(api):
    a, b = _mat(api, 8, 8, 1), _mat(api, 8, 8, 2)
    return api.matmul(api.matmul(a, b), api.matmul(b, a))


# ---- R7 -----------------------------------------------------------------------

@case("r7_golden")
def _(api):
    a = api.make_matrix(2, 1, "values", values=[1, 2])
    d = api.make_matrix(2, 2, "values", values=[3, 0, 0, 4])
    c = api.make_matrix(2, 1, "values", values=[5, 6])
    return api.as_scalar(api.matmul(api.matmul(api.transpose(a), api.diagmat(d)), c))


@case("r7_random")
def _(api):
    a, b, c = _mat(api, 20, 1, 1), _mat(api, 20, 20, 2), _mat(api, 20, 1, 3)
    return api.as_scalar(api.matmul(api.matmul(api.transpose(a), api.diagmat(b)), c))


@case("r7_fallback_computed_middle")
def _(api):
    a, b, c = _mat(api, 5, 1, 1), _mat(api, 5, 5, 2), _mat(api, 5, 1, 3)
    return api.as_scalar(api.matmul(api.matmul(api.transpose(a), api.diagmat(api.matmul(b, b))), c))


@case("as_scalar_dot")
def _(api):
    return api.as_scalar(api.matmul(_mat(api, 1, 4, 1), _mat(api, 4, 1, 2)))


# ---- R8 -------------------------------------------------------------------------

@case("r8_golden")
def _(api):
    a = api.make_matrix(2, 2, "values", values=[1, 3, 2, 4])
    return api.matmul(a, api.transpose(a))


@case("r8_rect")
def _(api):
    a = _mat(api, 9, 5, 1)
    return api.matmul(a, api.transpose(a))


@case("r8_transpose_left")
def _(api):
    a = _mat(api, 4, 6, 1)
    return api.matmul(api.transpose(a), api.leaf(a))


@case("r8_needs_identity")
def _(api):
    a = _mat(api, 5, 5, 1)
    return api.matmul(a, api.transpose(a.copy()))


# ---- R9 / R10 (structure scan at rewrite time) --------------------------------

@case("r9_diag_band", needs_scan=True)
def _(api):
    a = api.make_matrix(2, 2, "values", values=[2, 0, 0, 4])
    b = api.make_matrix(2, 1, "values", values=[2, 8])
    return api.matmul(api.inverse(a), b)


@case("r9_dense", needs_scan=True)
def _(api):
    return api.matmul(api.inverse(_host(api, _boosted(1, 8))), _mat(api, 8, 1, 2))


@case("r9_dense_multi_rhs", needs_scan=True)
def _(api):
    return api.matmul(api.inverse(_host(api, _boosted(3, 20))), _mat(api, 20, 3, 4))


@case("r9_inverse_on_right")
def _(api):
    return api.matmul(_mat(api, 4, 4, 2), api.inverse(_host(api, _boosted(1, 4))))


@case("r10_band", needs_scan=True)
def _(api):
    return api.solve(_host(api, _tridiag(1, 12)), _mat(api, 12, 1, 2))


@case("r10_triu", needs_scan=True)
def _(api):
    n = 10
    up = _rand(3, n, n)
    up[np.tril_indices(n, -1)] = 0.0
    up[np.diag_indices(n)] += n
    return api.solve(_host(api, up), _mat(api, n, 2, 4))


@case("r10_tril", needs_scan=True)
def _(api):
    n = 11
    lo = _rand(5, n, n)
    lo[np.triu_indices(n, 1)] = 0.0
    lo[np.diag_indices(n)] += n
    return api.solve(_host(api, lo), _mat(api, n, 2, 6))


@case("r10_sym", needs_scan=True)
def _(api):
    n = 9
    raw = _rand(5, n, n)
    sym = raw + raw.T
    sym[np.diag_indices(n)] += n
    return api.solve(_host(api, sym), _mat(api, n, 1, 6))


@case("r10_gen", needs_scan=True)
def _(api):
    return api.solve(_host(api, _boosted(7, 7)), _mat(api, 7, 1, 8))


@case("r10_runtime_sym")
def _(api):
    a, b = _mat(api, 10, 10, 3), _mat(api, 10, 1, 4)
    return api.solve(api.matmul(a, api.transpose(a)), b)


@case("r10_runtime_band")
def _(api):
    d = _host(api, np.arange(1.0, 7.0).reshape(6, 1) + 5.0)
    return api.solve(api.add(api.diagmat(d), api.diagmat(d)), _mat(api, 6, 2, 9))


@case("r10_runtime_gen")
def _(api):
    a = _host(api, _boosted(11, 8))
    return api.solve(api.smul(2.0, a), _mat(api, 8, 1, 12))


@case("inverse_plain")
def _(api):
    return api.inverse(_host(api, _boosted(4, 6)))


@case("solve_of_inverse_times", needs_scan=True)
def _(api):
    a = _host(api, _boosted(5, 6))
    b = _mat(api, 6, 6, 6)
    return api.matmul(api.matmul(api.inverse(a), b), _mat(api, 6, 1, 7))


# ---- mixed ----------------------------------------------------------------------

@case("mixed_elementwise_of_products")
def _(api):
    a, b, c = _mat(api, 7, 7, 1), _mat(api, 7, 7, 2), _mat(api, 7, 7, 3)
    return api.sub(api.add(api.matmul(a, b), api.smul(2.0, api.matmul(b, c))), api.transpose(c))


@case("diagmat_plain")
def _(api):
    return api.diagmat(_mat(api, 5, 5, 3))


@case("diagmat_vector")
def _(api):
    return api.diagmat(_mat(api, 1, 5, 3))


# The ten canonical bench expressions (reference bench.py:76-130) at the
# sizes of the reference acceptance test; operand generation is part of
# the API being mirrored.
for _eid in range(1, 11):
    for _size in (4, 16, 50):
        def _bench_case(api, eid=_eid, size=_size):
            return api.build_expression(eid, size, 0)[0]
        CASES[f"bench_{_eid}_{_size}"] = _bench_case
        if _eid in (9, 10):
            NEEDS_SCAN.add(f"bench_{_eid}_{_size}")
