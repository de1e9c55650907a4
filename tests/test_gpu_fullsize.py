"""Parity at the BASELINE sizes, not just at small shapes.

Int64 offsets, grid limits, split-K choices and persistent-loop tails only
change at full scale, so every config is checked against the oracle
(oracle/lm_oracle.c, pinned bitwise to the reference) on its own seeded
inputs at the size the bench times:

* config 1 at 4096^2: the fused program bitwise;
* config 3c at 16384 x 2048: 16 sampled 64 x 64 output tiles (diagonal,
  edge, split-K boundary) against the oracle's gemm over all 16384 inner
  terms, and the whole output bitwise symmetric;
* config 4a at 8192: the exact-order LU's (mode "exact") factors, pivots
  and solution bitwise against digests of the oracle's run
  (tests/golden/lu8192.json, made by tests/golden/make_lu8192.py -- the
  oracle needs minutes); the default tensor-core LU against the residual
  bound and the oracle's pivots;
* config 5a: the seeded 262144-instance scheme, 256 instances per size
  class spread over the whole class (both ends: the persistent loops'
  tail), regenerated on the host with numpy;
* config 5b at world size 1: a 32768-wide row block through the planner
  and ShardedTrace vs the oracle.
"""

import hashlib
import json
import pathlib

import numpy as np
import pytest
import torch

import paper_2502_03000_b200 as lm
from oracle import lm_oracle as O
from paper_2502_03000_b200 import kernels as K
from paper_2502_03000_b200.batch import atb_schur_trace, empty_batch
from paper_2502_03000_b200.datagen import (batch_sizes, fill_batch_class, fill_seeded, host_batch_instance,
                                           host_draws, seed_for)
from paper_2502_03000_b200.matrix import fortran_empty

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def bits_equal(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.int64), y.view(np.int64))


def normwise(x, y):
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


def seeded_device(config, k, rows, cols):
    return fill_seeded(fortran_empty(rows, cols), seed_for(config, k))


def seeded_host(config, k, rows, cols):
    return np.asfortranarray(np.random.default_rng(seed_for(config, k)).uniform(-1.0, 1.0, (rows, cols)))


def test_config1_full_size_bitwise():
    n = 4096
    A, B, C = (seeded_device(1, k, n, n) for k in range(3))
    a, b, c = (lm.DenseMatrix(t) for t in (A, B, C))
    D = lm.evaluate(2 * a + b % c - a / (1 + abs(b))).to_numpy()
    h = [seeded_host(1, k, n, n) for k in range(3)]
    assert bits_equal(A.cpu().numpy(), h[0])  # the device generator is numpy's stream
    ops, args, *_ = K.parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
    ref = np.empty((n, n), order="F")
    O.program(ops.numpy(), args.numpy(), [2.0, 1.0], h, ref)
    assert bits_equal(D, ref)


def test_config3c_syrk_full_size_sampled_tiles():
    M, N = 16384, 2048
    A = seeded_device(3, 20, M, N)
    S = lm.evaluate(lm.DenseMatrix(A).t() * lm.DenseMatrix(A)).data
    assert torch.equal(S, S.t())  # mirrored bitwise
    Sh = S.cpu().numpy()
    Ah = A.cpu().numpy()
    starts = [0, 64, 1024 - 64, 1024, N - 64]  # first / second tiles, a split boundary, the last tile
    tiles = [(i, j) for i in starts for j in starts if i <= j][:16]
    for i0, j0 in tiles:
        ref = np.zeros((64, 64), order="F")
        O.gemm(Ah[:, i0:i0 + 64].T, Ah[:, j0:j0 + 64], ref)
        assert normwise(Sh[i0:i0 + 64, j0:j0 + 64], ref) <= 1e-12, (i0, j0)


@pytest.mark.slow
def test_config4a_exact_lu_full_size_bitwise():
    gold = json.loads((GOLDEN / "lu8192.json").read_text())
    n, k = gold["n"], gold["nrhs"]
    A = seeded_device(4, 0, n, n)
    A.diagonal().add_(float(n))
    b = seeded_device(4, 1, n, k)
    from paper_2502_03000_b200 import _native as N
    lu, piv = K.lu_factor(A, mode="exact")  # bitwise: the exact reference order
    x = b.clone()
    N.call("lm_lu_solve", 0, N.view(lu.data), piv.data_ptr(), N.view(x))

    def digest(t):
        return hashlib.sha256(np.asfortranarray(t.cpu().numpy()).tobytes(order="F")).hexdigest()
    assert digest(piv.to(torch.int64)) == gold["piv_sha256"]
    assert digest(lu.data) == gold["lu_sha256"]
    assert digest(x) == gold["x_sha256"]


def test_config4a_tensor_lu_full_size_residual_and_pivots():
    """The default (tensor-core trailing update) LU at 8192 on the bench's
    inputs: pivots equal the oracle's (digest), scaled residual <= 1e-10."""
    gold = json.loads((GOLDEN / "lu8192.json").read_text())
    n, k = gold["n"], gold["nrhs"]
    A = seeded_device(4, 0, n, n)
    A.diagonal().add_(float(n))
    b = seeded_device(4, 1, n, k)
    lu, piv = K.lu_factor(A, mode="tensor")
    assert hashlib.sha256(np.ascontiguousarray(piv.cpu().numpy()).tobytes()).hexdigest() == gold["piv_sha256"]
    x = b.clone()
    K.lu_solve_into(A, x)  # auto -> tensor at this size
    Ah, bh, xh = A.cpu().numpy(), b.cpu().numpy(), x.cpu().numpy()
    res = np.linalg.norm(Ah @ xh - bh, np.inf) / (np.linalg.norm(Ah, np.inf) * np.linalg.norm(xh, np.inf) +
                                                 np.linalg.norm(bh, np.inf))
    assert res <= 1e-10


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config5a_seeded_batch_sampled(dtype):
    """The bench's own inputs: 262144 instances, sizes from the seeded
    draw, each class generated chunk by chunk; 256 instances per class
    (spread over the whole class) against the oracle."""
    sizes = batch_sizes(262144)
    ops, args, *_ = K.parse_program("x0 x1 x2 * +")
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    for n in (32, 64, 128):
        count = int((sizes == n).sum())
        ops_dev = [fill_batch_class(empty_batch(count, n, n, dtype), k, n, 0) for k in range(4)]
        E, s = atb_schur_trace(*ops_dev)
        idx = sorted(set(np.linspace(0, count - 1, 252).round().astype(int).tolist()) | {0, 1, count - 2, count - 1})
        Ed, sd = E[idx].double().cpu().numpy(), s[idx].double().cpu().numpy()
        A0 = ops_dev[0][idx[-1]].double().cpu().numpy()
        want = host_batch_instance(0, n, idx[-1])
        if dtype == torch.float32:
            want = want.astype(np.float32).astype(np.float64)
        assert bits_equal(A0, want)  # the chunked device generator == numpy
        for t, i in enumerate(idx):
            A, B, C, D = (host_batch_instance(k, n, i) for k in range(4))
            if dtype == torch.float32:
                A, B, C, D = (np.asfortranarray(x.astype(np.float32).astype(np.float64)) for x in (A, B, C, D))
            g = np.zeros((n, n), order="F")
            O.gemm(A.T, B, g)
            Er = np.zeros((n, n), order="F")
            O.program(ops.numpy(), args.numpy(), [], [g, C, D], Er)
            tr = O.trace_of_product(A, B)
            assert normwise(Ed[t], Er) <= tol, (n, i)
            assert abs(sd[t] - tr) <= tol * max(abs(tr), np.sum(np.abs(A * B.T)) * 1e-2), (n, i)
        del ops_dev, E, s
        torch.cuda.empty_cache()


def test_config5b_row_block_world1():
    """A 256-row block of the 32768^2 problem through the planner and
    ShardedTrace (world size 1: the all-reduce is the identity)."""
    from paper_2502_03000_b200.shard import ShardedTrace
    n, r, lo = 32768, 256, 12288
    seeds = [seed_for(5, 50 + k) for k in range(3)]
    blk = [fill_seeded(fortran_empty(r, n), s, skip=lo * n, row_stream=n) for s in seeds]
    bc = fill_seeded(fortran_empty(n, r), seeds[1], skip=lo, row_stream=n)
    a, b, c = (lm.DenseMatrix(t) for t in blk)
    D = lm.evaluate(2 * a + b % c - a / (1 + abs(b))).to_numpy()
    h = [t.cpu().numpy() for t in blk]
    assert bits_equal(h[0][3], host_draws(seeds[0], (lo + 3) * n, n))  # row 12291 of A
    bch = bc.cpu().numpy()
    assert bits_equal(bch[5, :], host_draws(seeds[1], 5 * n + lo, r))  # B[5, lo:lo+r]
    ops, args, *_ = K.parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
    ref = np.empty((r, n), order="F")
    O.program(ops.numpy(), args.numpy(), [2.0, 1.0], [np.asfortranarray(x) for x in h], ref)
    assert bits_equal(D, ref)
    s = ShardedTrace()(blk[0], bc)
    tr = O.trace_of_product(np.asfortranarray(h[0]), np.asfortranarray(bch))
    assert abs(float(s.item()) - tr) <= 1e-12 * abs(tr)


def test_nccl_allreduce_through_the_c_abi_world1():
    """The 5b finish: lm_nccl_init_rank + lm_allreduce_sum_f64 (world size 1:
    the sum over one rank is the identity, but the NCCL calls run)."""
    import ctypes
    from paper_2502_03000_b200 import _native as N
    from paper_2502_03000_b200.shard import NcclComm
    ver = ctypes.c_int(0)
    N.check(N.load_library().lm_nccl_load(None, ctypes.byref(ver)), "lm_nccl_load")
    assert ver.value >= 22700
    comm = NcclComm()
    t = torch.tensor([3.25, -1.5], dtype=torch.float64, device="cuda")
    comm.allreduce_sum(t)
    assert t.cpu().tolist() == [3.25, -1.5]
    s = torch.tensor([2.0], dtype=torch.float64, device="cuda")
    N.call("lm_allreduce_sum_f64", comm._comm, s.data_ptr())
    assert float(s.item()) == 2.0
    comm.close()
