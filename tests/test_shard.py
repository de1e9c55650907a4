"""Row-sharded evaluation logic on CPU: world size 2 over gloo.

The partial trace of each rank is computed by the C oracle (standing in
for the device kernel, which needs a GPU); the test checks the row
partition and that partials + the all-reduce reproduce the full trace
on every rank, exactly as the GPU path composes them."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_03000_b200.shard import ShardedTrace, row_range


def test_row_range_partitions_exactly():
    for n in (1, 7, 8, 100, 32768):
        for g in (1, 2, 3, 4, 8):
            rngs = [row_range(n, r, g) for r in range(g)]
            assert rngs[0][0] == 0 and rngs[-1][1] == n
            assert all(rngs[i][1] == rngs[i + 1][0] for i in range(g - 1))
            sizes = [hi - lo for lo, hi in rngs]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import lm_oracle as O
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.uniform(-1, 1, (n, n)))
    B = np.asfortranarray(rng.uniform(-1, 1, (n, n)))
    lo, hi = row_range(n, rank, world)

    def oracle_partial(a_rows, b_cols, out):
        out[0] = O.trace_of_product(np.asfortranarray(a_rows.numpy()), np.asfortranarray(b_cols.numpy()))

    st = ShardedTrace(partial_fn=oracle_partial)
    out = st(torch.from_numpy(A[lo:hi, :].copy()), torch.from_numpy(B[:, lo:hi].copy()),
             torch.zeros(1, dtype=torch.float64))
    q.put((rank, float(out[0]), O.trace_of_product(A, B)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_trace_two_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 37, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    vals = {r: v for r, v, _ in res}
    full = res[0][2]
    assert len(vals) == world
    assert vals[0] == vals[1]  # every rank ends with the same all-reduced value
    assert abs(vals[0] - full) <= 1e-12 * max(abs(full), 1.0)
