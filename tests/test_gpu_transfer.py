"""Asynchronous uploads / downloads: results identical to synchronous
evaluation, and evaluation never reads an operand before its upload ends."""

import numpy as np
import pytest
import torch

import paper_2502_03000_b200 as lm

pytestmark = pytest.mark.gpu


def _pin(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory().t()


def test_upload_evaluate_download_bitwise():
    rng = np.random.default_rng(7)
    a, b = rng.uniform(-1, 1, (1500, 1200)), rng.uniform(-1, 1, (1500, 1200))
    v = rng.uniform(-1, 1, (1500, 1))
    A, B, V = lm.upload(_pin(a)), lm.upload(_pin(b)), lm.upload(_pin(v))
    r = lm.download(lm.evaluate(lm.diagmat(V) * B + A)).wait()
    ref = lm.evaluate(lm.diagmat(lm.DenseMatrix(v)) * lm.DenseMatrix(b) + lm.DenseMatrix(a)).to_numpy()
    assert np.array_equal(r.numpy(), ref)
    t = lm.download(lm.evaluate(lm.trace(A * B.t()), host_scalar=False)).wait()
    assert float(t[0, 0]) == lm.evaluate(lm.trace(lm.DenseMatrix(a) * lm.DenseMatrix(b).t()))


def test_evaluation_waits_for_a_large_upload():
    """A 512 MB upload followed at once by an evaluation and a structure scan."""
    rng = np.random.default_rng(8)
    n = 8192
    a = rng.uniform(-1, 1, (n, n))
    A = lm.upload(_pin(a))
    s = lm.evaluate(lm.trace(A * A), host_scalar=True)
    ref = float(np.sum(a * a.T))
    assert abs(s - ref) <= 1e-12 * float(np.sum(np.abs(a) * np.abs(a.T)))
    B = lm.upload(_pin(np.triu(a)))
    info = lm.analyze_structure(B)
    assert info.lower_bandwidth == 0 and info.is_upper_triangular


def test_chunked_pipeline_matches_eager():
    """Column-chunked uploads into one device matrix, evaluation on column
    views as chunks arrive, downloads into pinned slices (bench config 2's
    end-to-end path)."""
    from paper_2502_03000_b200.matrix import MatrixView
    rng = np.random.default_rng(9)
    n, K = 1024, 8
    w = n // K
    a, b, v = rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, 1))
    pA, pB, pv = _pin(a), _pin(b), _pin(v)
    o2 = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
    o3 = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
    V = lm.upload(pv)
    A, B = lm.empty_matrix(n, n), lm.empty_matrix(n, n)
    fs = []
    for k in range(K):
        lm.upload_into(B, pB[:, k * w:(k + 1) * w], k * w)
        fs.append(lm.download(lm.evaluate(lm.diagmat(V) * MatrixView(B, 0, k * w, n, w)),
                              out=o2[:, k * w:(k + 1) * w]))
    for k in range(K):
        lm.upload_into(A, pA[:, k * w:(k + 1) * w], k * w)
        fs.append(lm.download(lm.evaluate(MatrixView(A, 0, k * w, n, w) * lm.diagmat(MatrixView(V, k * w, 0, w, 1))),
                              out=o3[:, k * w:(k + 1) * w]))
    t = lm.download(lm.evaluate(lm.trace(A * B), host_scalar=False))
    for f in fs:
        f.wait()
    Ad, Bd, Vd = lm.DenseMatrix(a), lm.DenseMatrix(b), lm.DenseMatrix(v)
    assert np.array_equal(o2.numpy(), lm.evaluate(lm.diagmat(Vd) * Bd).to_numpy())
    assert np.array_equal(o3.numpy(), lm.evaluate(Ad * lm.diagmat(Vd)).to_numpy())
    assert float(t.wait()[0, 0]) == lm.evaluate(lm.trace(Ad * Bd))
