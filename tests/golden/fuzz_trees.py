"""Seeded random expression trees over a small set of leaf shapes, built
through whichever API module is passed in (the reference ``lazymat`` when
making goldens, this package in the tests).  Shapes conform or not at
random, so validation errors, their messages and error paths are
exercised as well as shape inference and rendering."""

import random

LEAF_SHAPES = [(4, 4), (4, 1), (1, 4), (1, 1), (4, 3), (3, 4), (3, 3), (3, 1)]


def _values(r, c):
    """Seeded U(-1,1) values (column-major), square leaves boosted by 4 on
    the diagonal so inverses and solves are well defined."""
    import numpy as np
    v = np.random.default_rng(10 * r + c).uniform(-1.0, 1.0, (r, c))
    if r == c:
        v = v + 4.0 * np.eye(r)
    return [float(x) for x in v.flatten(order="F")]


def leaves(api):
    return [api.make_matrix(r, c, fill="values", values=_values(r, c)) for r, c in LEAF_SHAPES]


def build(api, mats, rng: random.Random, depth: int):
    if depth == 0 or rng.random() < 0.25:
        return api.leaf(mats[rng.randrange(len(mats))])
    op = rng.randrange(12)
    a = build(api, mats, rng, depth - 1)
    if op == 0:
        return api.add(a, build(api, mats, rng, depth - 1))
    if op == 1:
        return api.sub(a, build(api, mats, rng, depth - 1))
    if op == 2:
        return api.matmul(a, build(api, mats, rng, depth - 1))
    if op == 3:
        return api.smul(rng.choice([0.5, -2.0, 3.0]), a)
    if op == 4:
        return api.transpose(a)
    if op == 5:
        return api.inverse(a)
    if op == 6:
        return api.solve(a, build(api, mats, rng, depth - 1))
    if op == 7:
        return api.diagmat(a)
    if op == 8:
        return api.trace(a)
    if op == 9:
        return api.as_scalar(a)
    if op == 10:
        return api.col_of(a, rng.randrange(5))
    return api.row_of(a, rng.randrange(5))


def trees(api, n_trees: int = 400, seed: int = 2025):
    rng = random.Random(seed)
    mats = leaves(api)
    return [build(api, mats, rng, rng.randrange(1, 5)) for _ in range(n_trees)]


def value_record(api, t):
    """The evaluate() result as a flat column-major list (or [float]), or
    the error type name."""
    try:
        v = api.evaluate(t)
    except Exception as e:  # noqa: BLE001
        return ["error", type(e).__name__]
    if isinstance(v, float):
        return ["ok", [v]]
    return ["ok", [float(x) for x in v.to_values()]]


def record(api, n_trees: int = 400, seed: int = 2025):
    """[(render, shape-or-error)] for n_trees seeded trees."""
    out = []
    for t in trees(api, n_trees, seed):
        try:
            sh = api.validate(t)
            ish = api.infer_shape(t)
            res = ["ok", [int(sh.n_rows), int(sh.n_cols), bool(sh.is_scalar)], str(ish)]
        except Exception as e:  # noqa: BLE001 -- the error type and message are the record
            res = ["error", type(e).__name__, str(e)]
        out.append([api.render_expr(t), res])
    return out
