"""Generate golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``lazymat`` from /root/reference/pkg/src (read-only: numba's
on-disk cache is redirected to /tmp and bytecode writing is disabled so
nothing is written into the reference tree) and records

* kernels.npz / kernels.json -- inputs and outputs of every reference
  ``_loops`` function (the drop-in seam) on seeded
  inputs, including strided views and edge shapes.  They pin the C
  oracle (oracle/lm_oracle.c) bit-for-bit.
* plans.json / plans.npz -- for every case in tests/golden/cases.py: the
  reference plan (rule log, kernel sequence, params, slot shapes,
  describe() with storage ids normalised), the traced event stream and
  counters, and the evaluate()/naive_evaluate() results.

The fixtures are committed; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import json
import os
import pathlib
import re
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "lm_numba_cache"))
sys.dont_write_bytecode = True

HERE = pathlib.Path(__file__).resolve().parent
REF_SRC = pathlib.Path("/root/reference/pkg/src")

import numpy as np  # noqa: E402


def _import_reference():
    sys.path.insert(0, str(REF_SRC))
    import lazymat  # noqa: F401
    from lazymat import _loops
    return lazymat, _loops


_ID_RE = re.compile(r"\bm(\d+)\b")
_EV_ID_RE = re.compile(r"id=(\d+)")


def normalise_ids(text: str, pattern=_ID_RE, fmt="m#{}") -> str:
    """Replace storage ids by first-occurrence ordinals."""
    seen: dict[str, int] = {}

    def sub(m):
        k = m.group(1)
        if k not in seen:
            seen[k] = len(seen) + 1
        return fmt.format(seen[k])

    return pattern.sub(sub, text)


def normalise_trace(text: str) -> str:
    return normalise_ids(text, _EV_ID_RE, "id=#{}")


# ---------------------------------------------------------------------------
# kernel-level goldens
# ---------------------------------------------------------------------------

def kernel_goldens(_loops):
    rng = np.random.default_rng(20250203)
    arrays: dict[str, np.ndarray] = {}
    manifest: list[dict] = []

    def F(a):
        return np.asfortranarray(np.asarray(a, dtype=np.float64))

    def add(kind, idx, **kw):
        rec = {"kind": kind, "name": f"{kind}/{idx}"}
        for k, v in kw.items():
            if isinstance(v, np.ndarray):
                key = f"{kind}/{idx}/{k}"
                arrays[key] = v
                rec[k] = key
            else:
                rec[k] = v
        manifest.append(rec)

    # analyze -- sparse random patterns, square and rectangular
    for idx in range(60):
        n = int(rng.integers(1, 14))
        m = n if rng.random() < 0.7 else int(rng.integers(1, 14))
        a = rng.normal(size=(n, m))
        a[rng.random(size=(n, m)) < 0.6] = 0.0
        if idx % 7 == 0 and n == m:
            a = a + a.T
        a = F(a)
        lbw, ubw, sym = _loops._analyze(a, n == m)
        add("analyze", idx, a=a, square=bool(n == m), lbw=int(lbw), ubw=int(ubw), sym=bool(sym))

    # fused -- 1..6 terms, plus a transposed-view source
    for idx, nterm in enumerate([1, 2, 3, 4, 5, 6, 3]):
        r, c = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        srcs = [F(rng.uniform(-1, 1, (r, c))) for _ in range(nterm)]
        transposed = idx == 6
        if transposed:
            srcs[1] = np.ascontiguousarray(rng.uniform(-1, 1, (c, r))).T  # C-order .T view
        coeffs = [float(x) for x in rng.uniform(-3, 3, nterm)]
        out = np.zeros((r, c), order="F")
        if nterm == 1:
            _loops._fused1(coeffs[0], srcs[0], out)
        elif nterm == 2:
            _loops._fused2(coeffs[0], srcs[0], coeffs[1], srcs[1], out)
        elif nterm == 3:
            _loops._fused3(coeffs[0], srcs[0], coeffs[1], srcs[1], coeffs[2], srcs[2], out)
        elif nterm == 4:
            _loops._fused4(coeffs[0], srcs[0], coeffs[1], srcs[1], coeffs[2], srcs[2],
                           coeffs[3], srcs[3], out)
        else:
            _loops._fused1(coeffs[0], srcs[0], out)
            for k in range(1, nterm):
                _loops._fused_axpy(coeffs[k], srcs[k], out)
        kw = {f"s{k}": np.array(s, order="F") for k, s in enumerate(srcs)}
        add("fused", idx, coeffs=coeffs, nterm=nterm, out=out, **kw)

    # gemm -- random shapes, some with C-order (transposed) operands
    for idx in range(20):
        p, q, r = (int(x) for x in rng.integers(1, 13, size=3))
        a = F(rng.uniform(-1, 1, (p, q)))
        b = F(rng.uniform(-1, 1, (q, r)))
        if idx % 4 == 1:
            a = np.ascontiguousarray(rng.uniform(-1, 1, (q, p))).T
        if idx % 4 == 2:
            b = np.ascontiguousarray(rng.uniform(-1, 1, (r, q))).T
        out = np.zeros((p, r), order="F")
        _loops._gemm(a, b, out)
        add("gemm", idx, a=np.array(a, order="F"), b=np.array(b, order="F"), out=out)

    # gemv both ways
    for idx in range(6):
        p, q = (int(x) for x in rng.integers(1, 17, size=2))
        a = F(rng.uniform(-1, 1, (p, q)))
        trans = bool(idx % 2)
        x = rng.uniform(-1, 1, p if trans else q)
        out = np.zeros(q if trans else p)
        (_loops._gemv_t if trans else _loops._gemv)(a, x, out)
        add("gemv", idx, a=a, x=x, out=out, trans=trans)

    # syrk -- including the transposed (R8 left-transpose) operand
    for idx in range(10):
        n, k = (int(x) for x in rng.integers(1, 15, size=2))
        a = F(rng.uniform(-1, 1, (n, k)))
        if idx % 3 == 2:
            a = F(rng.uniform(-1, 1, (k, n))).T  # .T of an F-order matrix
        out = np.zeros((n, n), order="F")
        _loops._syrk(a, out)
        add("syrk", idx, a=np.array(a, order="F"), out=out)

    # diag_scale left/right with contiguous and diagonal-strided d
    for idx in range(8):
        r, c = (int(x) for x in rng.integers(1, 10, size=2))
        b = F(rng.uniform(-1, 1, (r, c)))
        side = "left" if idx % 2 == 0 else "right"
        n = r if side == "left" else c
        d = rng.uniform(-1, 1, n)
        out = np.zeros((r, c), order="F")
        (_loops._diag_scale_left if side == "left" else _loops._diag_scale_right)(d, b, out)
        add("diag_scale", idx, d=d, b=b, side=side, out=out)

    # diag_of_product / trace_of_product
    for idx in range(10):
        p, q = (int(x) for x in rng.integers(1, 20, size=2))
        a = F(rng.uniform(-1, 1, (p, q)))
        b = F(rng.uniform(-1, 1, (q, p)))
        if idx % 3 == 1:
            b = np.ascontiguousarray(rng.uniform(-1, 1, (p, q))).T
        d = np.zeros(p)
        _loops._diag_of_product(a, b, d)
        t = float(_loops._trace_of_product(a, b))
        add("dotprod", idx, a=np.array(a, order="F"), b=np.array(b, order="F"), diag=d, trace=t)

    # triple_diag_dot
    for idx in range(5):
        n = int(rng.integers(1, 30))
        a, d, c = (rng.uniform(-1, 1, n) for _ in range(3))
        add("triple", idx, a=a, d=d, c=c, out=float(_loops._triple_diag_dot(a, d, c)))

    # lu_factor / lu_solve -- general (real pivoting), dominant, singular
    for idx in range(16):
        n = int(rng.integers(1, 24))
        a = F(rng.uniform(-1, 1, (n, n)))
        if idx % 4 == 3:
            a = F(a + n * np.eye(n))
        if idx == 5 and n >= 3:
            a[:, 1] = 0.0  # singular: column 1 zero
        lu = np.array(a, order="F")
        piv = np.zeros(n, dtype=np.int64)
        rc = int(_loops._lu_factor(lu, piv))
        m = int(rng.integers(1, 4))
        b = F(rng.uniform(-1, 1, (n, m)))
        x = np.array(b, order="F")
        if rc == 0:
            _loops._lu_solve_inplace(lu, piv, x)
        add("lu", idx, a=a, rc=rc, lu=lu, piv=piv, b=b, x=x)

    # band factor/solve
    for idx in range(12):
        n = int(rng.integers(4, 25))
        kl, ku = int(rng.integers(0, 4)), int(rng.integers(0, 4))
        a = rng.uniform(-1, 1, (n, n))
        i, j = np.indices((n, n))
        a[(i - j > kl) | (j - i > ku)] = 0.0
        if idx % 3 != 2:
            a[np.diag_indices(n)] += n
        a = F(a)
        ab = np.zeros((2 * kl + ku + 1, n), order="F")
        piv = np.zeros(n, dtype=np.int64)
        _loops._pack_band(a, ab, kl, ku)
        rc = int(_loops._band_factor(ab, piv, kl, ku))
        b = F(rng.uniform(-1, 1, (n, 2)))
        x = np.array(b, order="F")
        if rc == 0:
            _loops._band_solve_inplace(ab, piv, x, kl, ku)
        add("band", idx, a=a, kl=kl, ku=ku, rc=rc, piv=piv, b=b, x=x)

    # triangular solves (incl. zero diagonal)
    for idx in range(8):
        n = int(rng.integers(1, 15))
        upper = bool(idx % 2 == 0)
        a = rng.uniform(-1, 1, (n, n))
        a = np.triu(a) if upper else np.tril(a)
        a[np.diag_indices(n)] += n
        if idx == 4:
            a[n // 2, n // 2] = 0.0
        a = F(a)
        b = F(rng.uniform(-1, 1, (n, 3)))
        x = np.array(b, order="F")
        rc = int(_loops._tri_solve_inplace(a, x, upper))
        add("tri", idx, a=a, upper=upper, rc=rc, b=b, x=x)

    # transpose_copy / diag_materialise
    for idx in range(4):
        r, c = (int(x) for x in rng.integers(1, 9, size=2))
        a = F(rng.uniform(-1, 1, (r, c)))
        out = np.zeros((c, r), order="F")
        _loops._transpose_copy(a, out)
        d = rng.uniform(-1, 1, r)
        dm = np.ones((r, r), order="F")
        _loops._diag_materialise(d, dm)
        add("copyops", idx, a=a, t=out, d=d, dm=dm)

    return arrays, manifest


# ---------------------------------------------------------------------------
# plan-level goldens
# ---------------------------------------------------------------------------

def _params_repr(params):
    return repr(tuple(params))


def plan_goldens(lm):
    sys.path.insert(0, str(HERE))
    from cases import CASES, NEEDS_SCAN  # noqa: E402

    arrays: dict[str, np.ndarray] = {}
    records = {}
    for name, build in CASES.items():
        tree = build(lm)
        plan = lm.rewrite(tree)
        rec = {
            "rule_log": list(plan.rule_log),
            "kernels": [s.kernel for s in plan.steps],
            "params": [_params_repr(s.params) for s in plan.steps],
            "dests": [list(plan.slot_shapes[s.dest]) for s in plan.steps],
            "slot_shapes": [list(s) for s in plan.slot_shapes],
            "result_slot": plan.result_slot,
            "scalar": bool(plan.scalar_result),
            "describe": normalise_ids(plan.describe()),
            "needs_scan": name in NEEDS_SCAN,
        }
        tr = lm.with_trace(lambda: lm.evaluate(tree))
        rec["trace"] = normalise_trace(lm.render_trace(tr.events))
        rec["counters"] = [tr.counters.flops, tr.counters.allocations, tr.counters.kernel_calls]
        res = tr.result
        if isinstance(res, float):
            rec["value"] = res
        else:
            arrays[f"{name}/evaluate"] = np.array(res.data, order="F")
        try:
            nv = lm.with_trace(lambda: lm.naive_evaluate(tree))
        except lm.LinalgError as exc:  # the reference's own behaviour, recorded as is
            rec["naive_error"] = type(exc).__name__
            records[name] = rec
            continue
        rec["naive_counters"] = [nv.counters.flops, nv.counters.allocations, nv.counters.kernel_calls]
        rec["naive_trace"] = normalise_trace(lm.render_trace(nv.events))
        if isinstance(nv.result, float):
            rec["naive_value"] = nv.result
        else:
            arrays[f"{name}/naive"] = np.array(nv.result.data, order="F")
        records[name] = rec
    return arrays, records


def main():
    lm, _loops = _import_reference()
    karr, kman = kernel_goldens(_loops)
    np.savez_compressed(HERE / "kernels.npz", **karr)
    (HERE / "kernels.json").write_text(json.dumps(kman, indent=0) + "\n")
    parr, prec = plan_goldens(lm)
    np.savez_compressed(HERE / "plans.npz", **parr)
    (HERE / "plans.json").write_text(json.dumps(prec, indent=1, sort_keys=True) + "\n")
    print(f"kernels: {len(kman)} cases, plans: {len(prec)} cases")


if __name__ == "__main__":
    main()
