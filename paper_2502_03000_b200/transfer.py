"""Asynchronous host <-> device transfers that overlap evaluation.

``upload(host)`` starts the host-to-device copy of a (pinned) host tensor
on a dedicated copy stream and returns the DenseMatrix at once; every
``evaluate``/``execute`` that reads the matrix makes the compute stream
wait for that copy (a stream-side event wait, not a host sync), so work on
other operands proceeds while it is in flight.  ``download(m)`` starts the
device-to-host copy of a result on a second copy stream after the work
queued so far on the compute stream, and returns a ``HostResult`` whose
``wait()`` blocks until the bytes have landed.  PCIe moves data in both
directions at once: a result of one expression can stream to the host
while the inputs of the next are still arriving.
"""

from __future__ import annotations

import torch

from .matrix import DenseMatrix, default_device, fortran_empty

__all__ = ["upload", "upload_into", "empty_matrix", "download", "HostResult", "wait_inputs"]

_streams: dict = {}


def _copy_streams(device):
    key = torch.device(device).index or 0
    if key not in _streams:
        with torch.cuda.device(key):
            _streams[key] = (torch.cuda.Stream(), torch.cuda.Stream())
    return _streams[key]


def upload(host: torch.Tensor, dtype=None) -> DenseMatrix:
    """Device copy of a 2-D host tensor (pinned for a truly asynchronous
    copy; any layout); the copy runs on the upload stream."""
    if host.dim() != 2:
        raise ValueError(f"upload needs a 2-D tensor, got {host.dim()}-D")
    dev = default_device()
    tdt = dtype or host.dtype
    out = fortran_empty(host.shape[0], host.shape[1], tdt, dev)
    h2d, _ = _copy_streams(dev)
    h2d.wait_stream(torch.cuda.current_stream(dev))  # `out` is allocated on the compute stream
    with torch.cuda.stream(h2d):
        out.copy_(host if host.dtype == tdt else host.to(tdt), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(h2d)
    # `out` belongs to the compute stream's pool: if the matrix is dropped
    # before any reader waited on the copy, the allocator must not hand the
    # block out again while the DMA is still writing it
    out.record_stream(h2d)
    m = DenseMatrix(out)
    m._ready = ev
    return m


def empty_matrix(rows: int, cols: int, dtype=torch.float64) -> DenseMatrix:
    """Uninitialised device matrix, e.g. the destination of chunked uploads."""
    return DenseMatrix(fortran_empty(rows, cols, dtype, default_device()))


def upload_into(dst: DenseMatrix, host: torch.Tensor, col0: int = 0) -> DenseMatrix:
    """Asynchronously copy a host block into columns [col0, col0 + w) of an
    existing device matrix (all rows).  Readers issued after this call wait
    for it (and for every earlier upload: the upload stream is in order), so
    a pipeline can compute on the columns that have arrived while the rest
    is still in flight."""
    if host.dim() != 2 or host.shape[0] != dst.n_rows or col0 < 0 or col0 + host.shape[1] > dst.n_cols:
        raise ValueError(f"upload_into: block {tuple(host.shape)} at column {col0} does not fit {dst.shape}")
    dev = dst.data.device
    h2d, _ = _copy_streams(dev)
    h2d.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(h2d):
        dst.data[:, col0:col0 + host.shape[1]].copy_(host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(h2d)
    dst.data.record_stream(h2d)  # as in upload(): no reuse while the DMA writes
    dst._ready = ev
    return dst


class HostResult:
    """A device-to-host copy in flight."""

    def __init__(self, tensor, event):
        self.tensor = tensor
        self.event = event

    def wait(self) -> torch.Tensor:
        self.event.synchronize()
        return self.tensor


def download(m, out: torch.Tensor | None = None) -> HostResult:
    """Copy a result DenseMatrix (or a 1x1 scalar result) to pinned host
    memory on the download stream, after everything queued so far on the
    compute stream."""
    data = m.data
    if out is None:
        out = torch.empty(data.shape[::-1], dtype=data.dtype).pin_memory().t()
    _, d2h = _copy_streams(data.device)
    d2h.wait_stream(torch.cuda.current_stream(data.device))
    with torch.cuda.stream(d2h):
        out.copy_(data, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(d2h)
    data.record_stream(d2h)  # the allocator must not reuse the buffer before the copy ends
    return HostResult(out, ev)


def wait_inputs(node) -> None:
    """Make the current stream wait for pending uploads of the tree's leaves."""
    stack = [node]
    cur = None
    while stack:
        n = stack.pop()
        if n.kind == "Leaf":
            m = n.value
            base = getattr(m, "base", m)
            ev = getattr(base, "_ready", None)
            if ev is not None:
                if cur is None:
                    cur = torch.cuda.current_stream(base.data.device)
                cur.wait_event(ev)
        else:
            stack.extend(n.children)
