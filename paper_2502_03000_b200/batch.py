"""Batched evaluation of many independent small expression instances.

The reference has no batch API (``evaluate`` takes one tree,
lazymat/rewrite.py:680-682; SURVEY.md finding 6).  These entry points
evaluate a batch of same-shaped instances with ONE kernel per plan step
instead of one Python evaluate per instance, with per-instance results
identical to evaluating every instance on its own:

* ``solve_batched(A, b)``: inverse(A_i)*b_i (BASELINE config 4b).  One
  kernel classifies every instance with the R9/R10 structure ladder
  (lazymat/rewrite.py:389-414) and solves it with a register-resident LU
  in the reference's exact operation order -- values and pivots
  bit-identical to per-instance lazymat -- and the host reads (class,
  info) once.  Band / triangular instances are then re-solved through the
  single-instance planner (their plan is not lu_solve).
* ``atb_schur_trace(A, B, C, D)``: E_i = A_i.T*B_i + C_i % D_i and
  s_i = trace(A_i*B_i) (BASELINE config 5a), one fused kernel per size
  class that reads every operand once.

Batched operands are (batch, rows, cols) device tensors whose instances
are column-major: element (b, i, j) at b*rows*cols + i + j*rows (torch
strides (rows*cols, 1, rows)); ``stack_fortran`` builds one from host
arrays.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _native as N
from .errors import KernelContractError, SingularMatrixError
from .matrix import DenseMatrix, default_device

__all__ = ["stack_fortran", "empty_batch", "solve_batched", "atb_schur_trace", "analyze_batched",
           "BatchSolveResult"]


def empty_batch(batch: int, rows: int, cols: int, dtype=torch.float64, device=None) -> torch.Tensor:
    device = default_device() if device is None else device
    return torch.empty((batch, cols, rows), dtype=dtype, device=device).transpose(1, 2)


def stack_fortran(arrs, dtype=torch.float64, device=None) -> torch.Tensor:
    """(batch, r, c) host array-like -> device batch, per-instance F-order."""
    a = np.asarray(arrs, dtype=np.float64 if dtype == torch.float64 else np.float32)
    host = torch.from_numpy(np.ascontiguousarray(np.transpose(a, (0, 2, 1))))
    device = default_device() if device is None else device
    return host.to(device).transpose(1, 2)


def _check_batch(t: torch.Tensor, name: str):
    if t.dim() != 3:
        raise KernelContractError(f"{name}: batched operand must be (batch, rows, cols)")
    b, r, c = t.shape
    st = t.stride()
    ok = st[0] == r * c and (r <= 1 or st[1] == 1) and (c <= 1 or st[2] == r)
    if not ok and b * r * c > 0:
        raise KernelContractError(f"{name}: instances must be contiguous column-major (strides {(r * c, 1, r)})")
    N._dev_check(t)


def analyze_batched(A: torch.Tensor) -> np.ndarray:
    """(batch, 3) int64 host array: lower bandwidth, upper bandwidth,
    symmetric flag of every square instance (exact device scan)."""
    _check_batch(A, "analyze_batched")
    b, n, _ = A.shape
    out = torch.empty((b, 3), dtype=torch.int64, device=A.device)
    N.call("lm_analyze_batched", N.dtype_code(A), n, b, A.data_ptr(), out.data_ptr())
    return out.cpu().numpy()


class BatchSolveResult:
    """x (batch, n, 1) device tensor, the per-instance structure class
    and the rule log the single-instance planner would record."""

    _TAGS = {0: ["R9"], 1: ["R9", "R10:BAND"], 2: ["R9", "R10:TRIU"], 3: ["R9", "R10:TRIL"],
             4: ["R9", "R10:SYM-DETECTED"]}

    def __init__(self, x, cls):
        self.x = x
        self.cls = cls  # 0 gen, 1 band, 2 triu, 3 tril, 4 sym (numpy int8)

    @property
    def lu_mask(self):
        return (self.cls == 0) | (self.cls == 4)

    @property
    def rule_logs(self):
        return [list(self._TAGS[int(c)]) for c in self.cls]


def _classify(info, n):
    """The reference ladder (lazymat/rewrite.py:146-173) per instance."""
    lbw, ubw, sym = info[:, 0], info[:, 1], info[:, 2].astype(bool)
    band = lbw + ubw <= max(4, n // 4)
    triu = ~band & (lbw == 0)
    tril = ~band & ~triu & (ubw == 0)
    symm = ~band & ~triu & ~tril & sym
    return band, triu, tril, symm


_PINNED = threading.local()


def _pinned_i32(count: int) -> torch.Tensor:
    """A reusable pinned host buffer (per thread) for the (class, info)
    read-back: a pageable .cpu() copy costs tens of microseconds more."""
    buf = getattr(_PINNED, "i32", None)
    if buf is None or buf.numel() < count:
        buf = torch.empty(max(count, 1 << 14), dtype=torch.int32, pin_memory=True)
        _PINNED.i32 = buf
    return buf[:count]


def solve_batched(A: torch.Tensor, b: torch.Tensor, *, check: bool = True) -> BatchSolveResult:
    """inverse(A_i) * b_i for every instance (R9 -> R10 dispatch -> solve).

    A: (batch, n, n), b: (batch, n, 1); both per-instance F-order.  A is
    not modified.  Raises SingularMatrixError naming the first failing
    instance when ``check`` (one host sync, as the reference raises
    synchronously)."""
    _check_batch(A, "solve_batched A")
    _check_batch(b, "solve_batched b")
    bt, n, n2 = A.shape
    if n != n2 or b.shape[1] != n or b.shape[2] != 1:
        raise KernelContractError("solve_batched: A must be (batch, n, n) and b (batch, n, 1)")
    x = torch.empty((bt, 1, n), dtype=A.dtype, device=A.device).transpose(1, 2)
    # b dense (batch*n consecutive elements, as _check_batch guarantees) and of x's type
    same = b.dtype == x.dtype and b.stride(0) == n and (n == 1 or b.stride(1) == 1)
    if n <= 64 and A.dtype == torch.float64:
        # one kernel: structure class + exact LU solve of every instance; one
        # host read of (class, info) into pinned memory; b is copied into x
        # inside the call (one cudaMemcpyAsync)
        if not same:
            x.copy_(b)
        src = b if same else x
        ci = torch.empty(2 * bt, dtype=torch.int32, device=A.device)
        N.call("lm_solve_batched_classified_from", N.dtype_code(A), n, bt, A.data_ptr(), src.data_ptr(),
               x.data_ptr(), ci.data_ptr(), ci.data_ptr() + 4 * bt)
        host_t = _pinned_i32(2 * bt)
        host_t.copy_(ci, non_blocking=True)
        torch.cuda.current_stream(A.device).synchronize()
        host = host_t.numpy()
        cls, hinfo = host[:bt], host[bt:]
        if not cls.any() and not hinfo.any():  # every instance general and solved (the common case)
            return BatchSolveResult(x, np.zeros(bt, dtype=np.int8))
        cls, hinfo = cls.astype(np.int8), hinfo.copy()
    else:
        if same:
            x.as_strided((x.numel(),), (1,)).copy_(b.as_strided((b.numel(),), (1,), b.storage_offset()))
        else:
            x.copy_(b)
        info = analyze_batched(A)
        band, triu, tril, symm = _classify(info, n)
        cls = np.zeros(bt, dtype=np.int8)
        cls[symm] = 4
        cls[tril] = 3
        cls[triu] = 2
        cls[band] = 1
        hinfo = None
    lu_mask = (cls == 0) | (cls == 4)
    if hinfo is not None and lu_mask.all():
        if check:
            bad = np.flatnonzero(hinfo)
            if bad.size:
                i = int(bad[0])
                col = int(hinfo[i]) - 1
                raise SingularMatrixError(f"singular matrix in instance {i}: zero pivot in column {col}",
                                          column=col)
        return BatchSolveResult(x, cls)
    # mixed classes (or n > 64): instances in index order; LU-class ones
    # were solved above, the others take the single-instance planner
    from .expr import inverse
    from .rewrite import evaluate
    for i in range(bt):
        if hinfo is not None and lu_mask[i]:
            if check and hinfo[i]:
                col = int(hinfo[i]) - 1
                raise SingularMatrixError(f"singular matrix in instance {i}: zero pivot in column {col}",
                                          column=col)
            continue
        ai = DenseMatrix(A[i])
        bi = DenseMatrix(b[i])
        x[i].copy_(evaluate(inverse(ai) * bi).data)
    return BatchSolveResult(x, cls)


def atb_schur_trace(A, B, C, D, out=None):
    """E_i = A_i.T @ B_i + C_i % D_i and s_i = trace(A_i @ B_i) for one
    size class (all instances n x n).  Returns (E, s); ``out=(E, s)``
    writes into caller-provided buffers (E per-instance F-order like the
    operands, s a contiguous vector)."""
    for t, nm in ((A, "A"), (B, "B"), (C, "C"), (D, "D")):
        _check_batch(t, f"atb_schur_trace {nm}")
    bt, n, n2 = A.shape
    if n != n2 or any(tuple(t.shape) != (bt, n, n) for t in (B, C, D)):
        raise KernelContractError("atb_schur_trace: all operands must be (batch, n, n)")
    if len({A.dtype, B.dtype, C.dtype, D.dtype}) != 1:
        raise KernelContractError("atb_schur_trace: operands must share one element type")
    if out is None:
        E = empty_batch(bt, n, n, A.dtype, A.device)
        s = torch.empty(bt, dtype=A.dtype, device=A.device)
    else:
        E, s = out
        _check_batch(E, "atb_schur_trace E")
        if tuple(E.shape) != (bt, n, n) or E.dtype != A.dtype:
            raise KernelContractError("atb_schur_trace: out E must be (batch, n, n) of the operands' type")
        if s.dim() != 1 or s.shape[0] != bt or s.dtype != A.dtype or (bt > 1 and s.stride(0) != 1):
            raise KernelContractError("atb_schur_trace: out s must be a contiguous (batch,) vector")
        N._dev_check(s)
    N.call("lm_expr_atb_schur_trace_batched", N.dtype_code(A), n, bt, A.data_ptr(), B.data_ptr(), C.data_ptr(),
           D.data_ptr(), E.data_ptr(), s.data_ptr())
    return E, s
