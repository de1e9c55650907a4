"""Whole-plan CUDA-graph capture in the executor.

``capture(expr_or_plan)`` runs the plan once eagerly (NVRTC programs are
compiled, the scratch pool is sized), then records ONE CUDA graph of
``execute`` -- every kernel of the plan, its temporaries (graph-private
memory) and the result buffer -- and returns a ``CapturedPlan`` whose call
replays it: one launch per evaluation instead of one per plan step, no
Python in the loop.  The leaves are read at replay time, so new inputs are
written into the same DenseMatrix buffers (``A.data.copy_(...)``) before a
replay (with ``upload_into`` the replay waits, stream-side, for the
copy when the graph was captured from a tree).  The result object is
reused (overwritten) by every replay.

Plans whose steps synchronise with the host cannot be captured: the solve
family reads the factorisation status to raise SingularMatrixError
(lazymat/kernels.py:194-198) and the runtime structure dispatch reads the
bandwidths (lazymat/rewrite.py:592-608); ``capture`` rejects them with
KernelContractError.
"""

from __future__ import annotations

import torch

from . import _native
from .errors import BackendUnavailableError, KernelContractError
from .expr import ExprNode
from .rewrite import Plan, execute, rewrite
from .transfer import wait_inputs

__all__ = ["CapturedPlan", "capture"]

_HOST_SYNC_KERNELS = {"lu_solve", "band_solve", "triangular_solve", "explicit_inverse"}


class CapturedPlan:
    """A plan recorded as one CUDA graph; call it to evaluate again."""

    def __init__(self, plan: Plan, warmup: int = 1, tree=None):
        syncing = sorted({st.kernel for st in plan.steps} & _HOST_SYNC_KERNELS)
        if syncing:
            raise KernelContractError(f"plan step(s) {syncing} synchronise with the host; not capturable")
        if not _native.cuda_available():
            raise BackendUnavailableError("CUDA-graph capture needs a CUDA device")
        self.plan = plan
        self.tree = tree  # when known: replays wait (stream-side) for uploads into its leaves
        torch.cuda.synchronize()  # pending uploads of the leaves (transfer.upload) have landed
        for _ in range(warmup):
            execute(plan, host_scalar=False)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            execute(plan, host_scalar=False)  # stream-side warm-up, as torch recommends before capture
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(self.graph):
            self.result = execute(plan, host_scalar=False)
        torch.cuda.synchronize()

    def replay(self) -> None:
        """Enqueue one evaluation on the current stream (no host sync)."""
        if self.tree is not None:
            wait_inputs(self.tree)
        self.graph.replay()

    def __call__(self, host_scalar: bool = True):
        self.replay()
        if self.plan.scalar_result and host_scalar:
            return float(self.result.data[0, 0].item())
        return self.result


def capture(expr: ExprNode | Plan, warmup: int = 1) -> CapturedPlan:
    """Rewrite (if given a tree) and capture the plan as one CUDA graph."""
    if isinstance(expr, Plan):
        return CapturedPlan(expr, warmup=warmup)
    return CapturedPlan(rewrite(expr), warmup=warmup, tree=expr)
