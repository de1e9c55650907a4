"""Seeded synthetic operands, generated in device memory.

SURVEY.md 8(d) fixes every BASELINE operand as a numpy fill:
``np.random.default_rng(seed).uniform(-1, 1, shape)`` in C order, then
stored column-major.  ``fill_seeded`` writes exactly those values (bit for
bit) straight into HBM with ``lm_fill_pcg64``: the 75 GB config-5a batch
takes milliseconds instead of minutes of host generation plus PCIe, and
the host can still check any element with numpy (``host_draws``: the
same generator advanced to the element's draw number).

Seed schemes used by the bench and the full-size parity tests:

* configs 1-4 and 5b: operand k of config c uses
  ``1000003*42 + 101*c + k`` (5b: k = 50 + operand index);
* config 5a: instance sizes from ``default_rng(1000003*42 + 101*5 + 99)
  .choice([32, 64, 128], 262144)``; operand k (A, B, C, D = 0..3) of the
  size-n class is generated in chunks of 4096 class instances, chunk q
  seeded with the entropy list ``[1000003*42 + 101*5 + k, n, q]``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N

__all__ = ["rng_state", "fill_seeded", "host_draws", "seed_for", "batch_chunk_seed", "CHUNK",
           "batch_sizes", "fill_batch_class", "host_batch_instance"]

BASE_SEED = 42
CHUNK = 4096  # instances per seeded chunk of a size class


def seed_for(config: int, k: int, seed: int = BASE_SEED) -> int:
    """Operand k of config c (the scheme of lazymat/bench.py:49-50)."""
    return 1000003 * seed + 101 * config + k


def batch_chunk_seed(k: int, n: int, q: int, seed: int = BASE_SEED) -> list:
    """SeedSequence entropy of chunk q of operand k of the size-n class (config 5a)."""
    return [seed_for(5, k, seed), n, q]


def batch_sizes(count: int = 262144, sizes=(32, 64, 128), seed: int = BASE_SEED) -> np.ndarray:
    """Per-instance sizes of config 5a, in instance order."""
    return np.random.default_rng(seed_for(5, 99, seed)).choice(np.asarray(sizes), count)


def rng_state(seed) -> tuple:
    """(state, inc) of np.random.default_rng(seed)'s PCG64 right after seeding."""
    st = np.random.default_rng(seed).bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise RuntimeError(f"numpy default_rng is {st['bit_generator']}, expected PCG64")
    return int(st["state"]["state"]), int(st["state"]["inc"])


def _u64(x: int):
    return (x >> 64) & 0xFFFFFFFFFFFFFFFF, x & 0xFFFFFFFFFFFFFFFF


def fill_seeded(t: torch.Tensor, seed, skip: int = 0, row_stream: int | None = None,
                inst_stream: int | None = None, lo: float = -1.0, hi: float = 1.0) -> torch.Tensor:
    """Fill a column-major device matrix (rows, cols) or batch (b, rows, cols)
    with draws of default_rng(seed).uniform(lo, hi): element (b, i, j) is
    draw ``skip + b*inst_stream + i*row_stream + j`` (defaults: rows*cols and
    cols, i.e. the C-order draws of one (b, rows, cols) numpy array)."""
    if t.dim() == 2:
        rows, cols = t.shape
        batch, bstride = 1, 0
        rs, ld = t.stride()
    elif t.dim() == 3:
        batch, rows, cols = t.shape
        bstride, rs, ld = t.stride()
    else:
        raise ValueError("fill_seeded: 2-D or 3-D tensor expected")
    if rows > 1 and rs != 1:
        raise ValueError("fill_seeded: column-major (unit row stride) storage expected")
    if cols <= 1:
        ld = max(ld, rows)
    state, inc = rng_state(seed)
    sh, sl = _u64(state)
    ih, il = _u64(inc)
    row_stream = cols if row_stream is None else row_stream
    inst_stream = rows * cols if inst_stream is None else inst_stream
    N.call("lm_fill_pcg64", N.dtype_code(t), t.data_ptr(), batch, rows, cols, ld, bstride, inst_stream, row_stream,
           int(skip), sh, sl, ih, il, float(lo), float(hi))
    return t


def host_draws(seed, start: int, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Draws [start, start + count) of default_rng(seed).uniform(lo, hi) on the host."""
    g = np.random.default_rng(seed)
    g.bit_generator.advance(int(start))
    return g.uniform(lo, hi, int(count))


def host_matrix(seed, rows: int, cols: int, skip: int = 0, row_stream: int | None = None) -> np.ndarray:
    """Host twin of fill_seeded for one matrix (F-order float64)."""
    row_stream = cols if row_stream is None else row_stream
    if row_stream == cols:
        return np.asfortranarray(host_draws(seed, skip, rows * cols).reshape(rows, cols))
    out = np.empty((rows, cols), order="F")
    for i in range(rows):
        out[i, :] = host_draws(seed, skip + i * row_stream, cols)
    return out


def fill_batch_class(t: torch.Tensor, k: int, n: int, first: int, seed: int = BASE_SEED) -> torch.Tensor:
    """Operand k of class-n instances [first, first + t.shape[0]) of config 5a
    into the (count, n, n) column-major batch t, chunk by chunk."""
    count = t.shape[0]
    i = 0
    while i < count:
        g = first + i
        q, pos = divmod(g, CHUNK)
        m = min(count - i, CHUNK - pos)
        fill_seeded(t[i:i + m], batch_chunk_seed(k, n, q, seed), skip=pos * n * n)
        i += m
    return t


def host_batch_instance(k: int, n: int, idx: int, seed: int = BASE_SEED) -> np.ndarray:
    """Operand k of class-n instance idx of config 5a (F-order float64, host)."""
    q, pos = divmod(idx, CHUNK)
    return host_matrix(batch_chunk_seed(k, n, q, seed), n, n, skip=pos * n * n)
