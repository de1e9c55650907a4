"""Row-sharded multi-GPU evaluation (BASELINE config 5b).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).
For an n x n problem, rank g of G owns rows [lo_g, hi_g) of every
operand (``row_range``: contiguous, balanced):

* element-wise expressions (the config-1 program) are row-local -- each
  rank evaluates its row block through the normal planner/kernels, no
  communication at all;
* trace(A*B) = sum_g sum_{i in rows_g} sum_k A[i,k] B[k,i]: rank g needs
  its row block of A and the matching COLUMN block of B, computes the
  partial with the same trace_of_product kernel (it accepts p x q / q x p
  operands, lazymat/kernels.py:157-164), and one NCCL all-reduce of a
  single float64 finishes it -- the only collective, because it is the
  only real exchange step.  The all-reduce goes through
  the C-ABI (lm_allreduce_sum_f64 on an lm_nccl_init_rank communicator,
  ``NcclComm``); torch.distributed only carries the 128-byte NCCL unique id
  from rank 0 to the others.

The partial-trace function is injectable so the host-side sharding and
reduction logic is testable on CPU with the gloo backend
(tests/test_shard.py: CPU tensors reduce through torch.distributed there);
the product path always uses the CUDA kernel and the library's NCCL.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import sys

import torch

from . import kernels
from .matrix import DenseMatrix

__all__ = ["row_range", "ShardedTrace", "NcclComm", "eval_rows", "fill_uniform", "partition_by_cost", "class_ranges"]


def row_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous balanced row block [lo, hi) of rank ``rank``."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def partition_by_cost(costs, world: int) -> list:
    """Contiguous instance ranges [(lo, hi)] per rank, balanced by cost.

    Independent instances (configs 4b, 5a) shard with no collective
    (SURVEY.md 8(e)): rank g takes the instances whose cumulative cost
    (realised n^3 per instance) falls in [g/G, (g+1)/G) of the total, so a
    fixed batch strong-scales and each rank's share of the work differs
    from 1/G by at most one instance.  Every instance lands on exactly one
    rank, in order."""
    import numpy as np
    c = np.asarray(costs, dtype=np.float64)
    if world < 1:
        raise ValueError("world must be >= 1")
    if c.size == 0:
        return [(0, 0)] * world
    cum = np.cumsum(c)
    total = cum[-1]
    # rank boundary g: the first instance whose cost MIDPOINT passes g/G
    mid = cum - c / 2
    cuts = [0] + [int(np.searchsorted(mid, total * g / world, side="left")) for g in range(1, world)] + [c.size]
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def class_ranges(sizes, lo: int, hi: int, classes) -> dict:
    """For instances [lo, hi) of a mixed-size batch: {n: (first, count)} --
    the contiguous range of size-class-n indices (the instance's rank among
    the class-n instances of the WHOLE batch) this slice covers."""
    import numpy as np
    sizes = np.asarray(sizes)
    out = {}
    for n in classes:
        is_n = sizes == n
        first = int(is_n[:lo].sum())
        out[n] = (first, int(is_n[lo:hi].sum()))
    return out


def _device_partial(a_rows: torch.Tensor, b_cols: torch.Tensor, out: torch.Tensor) -> None:
    kernels.trace_of_product(a_rows, b_cols, out=out)


def _dist_world(group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


@contextlib.contextmanager
def _stdout_to_stderr():
    """NCCL prints its version banner on file descriptor 1 at the first call
    (e.g. with NCCL_DEBUG=VERSION in the environment); keep the process's
    stdout -- bench.py's single JSON line -- clean by pointing fd 1 at
    stderr while NCCL initialises."""
    sys.stdout.flush()
    saved = os.dup(1)
    try:
        os.dup2(2, 1)
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


class NcclComm:
    """An NCCL communicator of the C-ABI (lm_nccl_init_rank), one process
    per GPU.  Rank 0 creates the unique id; with more than one rank it is
    broadcast over torch.distributed (rendezvous only -- no tensor data).
    Create it on every rank with the rank's device current."""

    def __init__(self, group=None):
        from . import _native as N
        self._N = N
        lib = N.load_library()
        self.rank, self.world = _dist_world(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            with _stdout_to_stderr():
                N.check(lib.lm_nccl_unique_id(uid), "lm_nccl_unique_id")
        if self.world > 1:
            import torch.distributed as dist
            box = [uid.raw if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        self._comm = ctypes.c_void_p()
        with _stdout_to_stderr():
            N.check(lib.lm_nccl_init_rank(self.world, self.rank, uid, ctypes.byref(self._comm)), "lm_nccl_init_rank")

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over the ranks, asynchronous on the current stream."""
        N = self._N
        N._dev_check(t)
        if not t.is_contiguous():
            raise ValueError("allreduce_sum: contiguous tensor expected")
        N.call("lm_allreduce_sum", self._comm, N.dtype_code(t), t.data_ptr(), t.numel())
        return t

    def close(self):
        if self._comm:
            self._N.check(self._N.load_library(False).lm_nccl_destroy(self._comm), "lm_nccl_destroy")
            self._comm = ctypes.c_void_p()

    def __del__(self):  # best effort
        try:
            self.close()
        except Exception:
            pass


class ShardedTrace:
    """trace(A @ B) over row shards: local partial + one all-reduce."""

    def __init__(self, group=None, partial_fn=None, comm: "NcclComm | None" = None):
        self.group = group
        self.partial_fn = partial_fn or _device_partial
        self.comm = comm

    def __call__(self, a_rows: torch.Tensor, b_cols: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
        """a_rows: (R, n) row block of A; b_cols: (n, R) matching column
        block of B.  Returns the 1-element tensor holding the GLOBAL trace
        (on every rank)."""
        if out is None:
            out = torch.empty(1, dtype=a_rows.dtype, device=a_rows.device)
        self.partial_fn(a_rows, b_cols, out)
        if out.is_cuda:
            if self.comm is None:  # created on first use, on every rank (collective rendezvous)
                self.comm = NcclComm(self.group)
            self.comm.allreduce_sum(out)
        elif _dist_world(self.group)[1] > 1:
            import torch.distributed as dist  # CPU partials (the gloo test of the sharding logic)
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)
        return out


def fill_uniform(t: torch.Tensor, seed: int, row0: int = 0, col0: int = 0, global_rows: int = None,
                 lo: float = -1.0, hi: float = 1.0) -> torch.Tensor:
    """Fill a device view with U(lo, hi) values that depend only on the
    GLOBAL element index (row0+i, col0+j): every rank generates its slices
    of one consistent distributed matrix (lm_fill_uniform)."""
    from . import _native as N
    if global_rows is None:
        global_rows = t.shape[0]
    N.call("lm_fill_uniform", N.dtype_code(t), N.view(t), int(seed) & 0xFFFFFFFFFFFFFFFF, int(row0), int(col0),
           int(global_rows), float(lo), float(hi))
    return t


def eval_rows(build, blocks: dict, lm_module=None):
    """Evaluate a row-local expression on this rank's row blocks through
    the ordinary planner: ``build(lm, mats)`` returns the tree; ``blocks``
    maps names to (R, n) device tensors (F-order)."""
    if lm_module is None:
        import paper_2502_03000_b200 as lm_module
    mats = {k: DenseMatrix(v) for k, v in blocks.items()}
    return lm_module.evaluate(build(lm_module, mats))
