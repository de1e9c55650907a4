"""Batched entry points vs per-instance oracle results."""

import numpy as np
import pytest
import torch

import paper_2502_03000_b200 as lm
from oracle import lm_oracle as O
from paper_2502_03000_b200.batch import atb_schur_trace, solve_batched, stack_fortran
from paper_2502_03000_b200.kernels import parse_program

pytestmark = pytest.mark.gpu


def bits_equal(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.int64), y.view(np.int64))


@pytest.mark.parametrize("n", [1, 7, 32, 64])
@pytest.mark.parametrize("kind", ["dominant", "general"])
def test_solve_batched_bitwise_vs_per_instance_reference(n, kind):
    rng = np.random.default_rng(n)
    bt = 37
    A = rng.uniform(-1, 1, (bt, n, n)) + (n * np.eye(n)[None] if kind == "dominant" else 0)
    b = rng.uniform(-1, 1, (bt, n, 1))
    res = solve_batched(stack_fortran(A), stack_fortran(b))
    x = res.x.cpu().numpy()
    for i in range(bt):
        rc, lu, piv = O.lu_factor(np.asfortranarray(A[i]))
        if n > 4 and kind == "general":
            pass
        xr = np.array(b[i], order="F")
        if rc == 0:
            O.lu_solve(lu, piv, xr)
        if res.lu_mask[i]:
            assert bits_equal(x[i], xr), i
        else:  # band/triangular instance: the single-instance plan result
            ref = lm.evaluate(lm.inverse(lm.DenseMatrix(A[i])) * lm.DenseMatrix(b[i])).to_numpy()
            assert bits_equal(x[i], ref)


@pytest.mark.parametrize("n", [1, 2, 8, 9, 15, 16, 17, 24, 31, 32, 33, 40, 48, 50, 57, 63, 64])
@pytest.mark.parametrize("with_lu", [False, True])
def test_lu_solve_batched_entry_bitwise(n, with_lu):
    """lm_lu_solve_batched (solve-only: the rolled shifted-row kernel; with
    LU output: the unrolled kernel): x and pivots bit-identical to the
    reference's _lu_factor + _lu_solve_inplace, general (pivoting) matrices
    and ties (repeated magnitudes) included."""
    from paper_2502_03000_b200 import _native as N

    rng = np.random.default_rng(1000 + n)
    bt = 29
    A = rng.uniform(-1, 1, (bt, n, n))
    A[1::4] = np.round(A[1::4] * 4) / 4          # many equal |values|: first-maximum tie rule
    A[2::4] += n * np.eye(n)[None]
    b = rng.uniform(-1, 1, (bt, n, 1))
    At = stack_fortran(A)
    x = torch.tensor(b[:, :, 0], device="cuda").contiguous()
    piv = torch.zeros((bt, n), dtype=torch.int64, device="cuda")
    info = torch.zeros(bt, dtype=torch.int32, device="cuda")
    lu = torch.zeros((bt, n, n), dtype=torch.float64, device="cuda") if with_lu else None
    N.call("lm_lu_solve_batched", 0, n, bt, At.data_ptr(), x.data_ptr(), lu.data_ptr() if with_lu else None,
           piv.data_ptr(), info.data_ptr())
    torch.cuda.synchronize()
    xs, ps, inf = x.cpu().numpy(), piv.cpu().numpy(), info.cpu().numpy()
    for i in range(bt):
        rc, lur, pr = O.lu_factor(np.asfortranarray(A[i]))
        assert inf[i] == rc, i
        if rc:
            continue
        assert np.array_equal(ps[i], pr), i
        xr = np.array(b[i], order="F")
        O.lu_solve(lur, pr, xr)
        assert bits_equal(xs[i], xr[:, 0]), i
        if with_lu:
            assert bits_equal(lu[i].cpu().numpy().reshape(n, n).T, lur), i


def test_solve_batched_rule_logs_match_single_instance_planner():
    rng = np.random.default_rng(3)
    n, bt = 16, 5
    A = rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None]
    A[1] = np.triu(A[1])
    A[2] = A[2] + A[2].T
    b = rng.uniform(-1, 1, (bt, n, 1))
    res = solve_batched(stack_fortran(A), stack_fortran(b))
    for i in range(bt):
        plan = lm.rewrite(lm.inverse(lm.DenseMatrix(A[i])) * lm.DenseMatrix(b[i]))
        assert res.rule_logs[i] == plan.rule_log


def test_solve_batched_singular_instance_raises():
    n, bt = 8, 4
    A = np.tile(np.eye(n), (bt, 1, 1)) * 3.0 + 0.1
    A[2][:, 3] = 0.0
    with pytest.raises(lm.SingularMatrixError):
        solve_batched(stack_fortran(A), stack_fortran(np.ones((bt, n, 1))))


@pytest.mark.parametrize("n", [1, 5, 32, 33, 64, 128])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_atb_schur_trace_vs_oracle(n, dtype):
    rng = np.random.default_rng(n)
    bt = 9
    ops = [rng.uniform(-1, 1, (bt, n, n)) for _ in range(4)]
    if dtype == torch.float32:
        ops = [o.astype(np.float32).astype(np.float64) for o in ops]  # oracle on the f32-rounded inputs
    E, s = atb_schur_trace(*(stack_fortran(o, dtype=dtype) for o in ops))
    E, s = E.cpu().numpy(), s.cpu().numpy()
    pops, pargs, *_ = parse_program("x0 x1 x2 * +")
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    for i in range(bt):
        A, B, C, D = (np.asfortranarray(o[i]) for o in ops)
        g = np.zeros((n, n), order="F")
        O.gemm(A.T, B, g)
        Er = np.zeros((n, n), order="F")
        O.program(pops.numpy(), pargs.numpy(), [], [g, C, D], Er)
        assert np.max(np.abs(E[i] - Er)) <= tol * max(np.max(np.abs(Er)), 1e-30)
        tr = O.trace_of_product(A, B)
        assert abs(s[i] - tr) <= tol * max(abs(tr), np.sum(np.abs(A * B.T)) * 1e-2)


@pytest.mark.parametrize("n", [32, 64, 128])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_atb_schur_trace_many_instances_per_cta(n, dtype):
    """Batches larger than the persistent grid: every CTA runs several
    instances, so the n = 128 kernel's overlapped epilogue (instance j's E
    finished during instance j+1's main loop) and its drain are exercised;
    sampled instances against the oracle."""
    rng = np.random.default_rng(7 * n)
    bt = 701  # odd: the paired n = 64 kernel's last pair has one instance
    ops = [rng.uniform(-1, 1, (bt, n, n)) for _ in range(4)]
    if dtype == torch.float32:
        ops = [o.astype(np.float32).astype(np.float64) for o in ops]
    E, s = atb_schur_trace(*(stack_fortran(o, dtype=dtype) for o in ops))
    E, s = E.cpu().numpy(), s.cpu().numpy()
    pops, pargs, *_ = parse_program("x0 x1 x2 * +")
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    for i in sorted({0, 1, 147, 148, 149, 295, 296, 297, 443, 444, 591, 592, 699, 700, int(rng.integers(0, bt))}):
        A, B, C, D = (np.asfortranarray(o[i]) for o in ops)
        g = np.zeros((n, n), order="F")
        O.gemm(A.T, B, g)
        Er = np.zeros((n, n), order="F")
        O.program(pops.numpy(), pargs.numpy(), [], [g, C, D], Er)
        assert np.max(np.abs(E[i] - Er)) <= tol * max(np.max(np.abs(Er)), 1e-30), i
        tr = O.trace_of_product(A, B)
        assert abs(s[i] - tr) <= tol * max(abs(tr), np.sum(np.abs(A * B.T)) * 1e-2), i


@pytest.mark.parametrize("n", [1, 3, 5, 16, 33, 64])
def test_classified_kernel_matches_structure_scan(n):
    """The one-pass classify+solve kernel assigns every instance the class
    the batched structure scan + R10 ladder gives."""
    from paper_2502_03000_b200 import _native as N
    from paper_2502_03000_b200.batch import _classify, analyze_batched

    rng = np.random.default_rng(100 + n)
    mats = []
    for kind in range(12):
        a = rng.uniform(-1, 1, (n, n)) + n * np.eye(n)
        if kind % 6 == 1:
            a = np.triu(np.tril(a, 1), -1)          # tridiagonal (band)
        elif kind % 6 == 2:
            a = np.triu(a)
        elif kind % 6 == 3:
            a = np.tril(a)
        elif kind % 6 == 4:
            a = a + a.T
        elif kind % 6 == 5:
            a[rng.integers(0, n), rng.integers(0, n)] = 0.0
        mats.append(a)
    A = stack_fortran(np.array(mats))
    bt = A.shape[0]
    x = torch.zeros((bt, 1, n), dtype=torch.float64, device=A.device).transpose(1, 2)
    ci = torch.empty(2 * bt, dtype=torch.int32, device=A.device)
    N.call("lm_solve_batched_classified", 0, n, bt, A.data_ptr(), x.data_ptr(), ci.data_ptr(), ci.data_ptr() + 4 * bt)
    got = ci[:bt].cpu().numpy()
    band, triu, tril, symm = _classify(analyze_batched(A), n)
    want = np.zeros(bt, dtype=np.int32)
    want[symm] = 4
    want[tril] = 3
    want[triu] = 2
    want[band] = 1
    assert np.array_equal(got, want)


@pytest.mark.parametrize("which", ["c", "d", "e"])
def test_misaligned_operands_take_the_generic_kernel(which):
    """C, D or E 8 bytes off the 32-byte alignment the vectorised kernels
    need (a view with a storage offset): the call must take the generic
    kernel (no misaligned-address fault) and still match the oracle."""
    from paper_2502_03000_b200 import _native
    from paper_2502_03000_b200.batch import atb_schur_trace
    n, bt = 64, 5
    rng = np.random.default_rng(21)
    hs = [rng.uniform(-1, 1, (bt, n, n)) for _ in range(4)]
    ops = [stack_fortran(h) for h in hs]
    k = "abcd".index(which) if which != "e" else None

    def shifted(h):  # same values, storage offset of one element
        flat = torch.empty(bt * n * n + 1, dtype=torch.float64, device="cuda")
        v = flat[1:].view(bt, n, n).transpose(1, 2)
        v.copy_(stack_fortran(h))
        return v
    if k is not None:
        ops[k] = shifted(hs[k])
        E, s = atb_schur_trace(*ops)
    else:
        E = shifted(np.zeros((bt, n, n)))
        s = torch.empty(bt, dtype=torch.float64, device="cuda")
        atb_schur_trace(*ops, out=(E, s))
    assert _native.last_variant() == "generic"
    Eh, sh = E.cpu().numpy(), s.cpu().numpy()
    for i in range(bt):
        A, B, C, D = (np.asfortranarray(h[i]) for h in hs)
        Er = A.T @ B + C * D
        assert np.max(np.abs(Eh[i] - Er)) <= 1e-12 * np.max(np.abs(Er))
        tr = O.trace_of_product(A, B)
        assert abs(sh[i] - tr) <= 1e-12 * max(abs(tr), 1.0)


def _batched_lu_vs_oracle(A, b):
    """lm_lu_solve_batched (solve only) vs the oracle's lu_factor + lu_solve:
    x bitwise, info equal; returns the number of systems checked."""
    from paper_2502_03000_b200 import _native as N

    bt, n, _ = A.shape
    x = torch.tensor(b[:, :, 0], device="cuda").contiguous()
    piv = torch.zeros((bt, n), dtype=torch.int64, device="cuda")
    info = torch.zeros(bt, dtype=torch.int32, device="cuda")
    N.call("lm_lu_solve_batched", 0, n, bt, stack_fortran(A).data_ptr(), x.data_ptr(), None, piv.data_ptr(),
           info.data_ptr())
    torch.cuda.synchronize()
    xs, ps, inf = x.cpu().numpy(), piv.cpu().numpy(), info.cpu().numpy()
    for i in range(bt):
        rc, lur, pr = O.lu_factor(np.asfortranarray(A[i]))
        assert inf[i] == rc, (i, inf[i], rc)
        if rc:
            continue
        assert np.array_equal(ps[i], pr), i
        xr = np.array(b[i], order="F")
        O.lu_solve(lur, pr, xr)
        assert bits_equal(xs[i], xr[:, 0]), i
    return bt


@pytest.mark.parametrize("n", [33, 40, 57, 64])
def test_lu_solve_batched_pivot_free_path_edges(n):
    """The pivot-free fast path (n in 33..64) certifies every quotient and
    proves identity pivots (|multiplier| < 1); whatever it cannot certify
    falls to the pivoting kernel.  Edge systems: magnitudes scaled by 2^-600
    / 2^600 (outside the certified exponent window), exact zeros in A and b,
    power-of-two entries (quotients on binade boundaries), a multiplier of
    exactly 1 (|a_ik| == |a_kk|: the reference keeps p = k, the fast path
    must hand over), dominant and general matrices mixed in one batch.  x,
    pivots and info bitwise vs the oracle."""
    rng = np.random.default_rng(4000 + n)
    bt = 24
    A = rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None]
    b = rng.uniform(-1, 1, (bt, n, 1))
    A[1] *= 2.0 ** -600
    b[1] *= 2.0 ** -600
    A[2] *= 2.0 ** 600
    A[3][np.abs(A[3]) < 0.3] = 0.0
    b[3][::3] = 0.0
    A[4] = np.round(A[4] * 4) / 4 + n * np.eye(n)           # quarter-integers: many exact quotients
    A[5] = 2.0 ** np.round(rng.uniform(-4, 4, (n, n)))      # powers of two, then dominant
    A[5] += (2.0 * n * 16) * np.eye(n)
    A[6][1, 0] = A[6][0, 0]                                 # |l_10| == 1 exactly
    A[7] = rng.uniform(-1, 1, (n, n))                       # general: pivoting
    A[8] = np.triu(A[8])
    b[9] = 0.0
    assert _batched_lu_vs_oracle(A, b) == bt


def test_lu_solve_batched_default_is_pivot_free_kernel():
    from paper_2502_03000_b200 import _native as N

    rng = np.random.default_rng(5)
    n, bt = 64, 3
    A = rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None]
    _batched_lu_vs_oracle(A, rng.uniform(-1, 1, (bt, n, 1)))
    assert N.last_variant() == "nopiv64"
