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


# ---- instance partition of the batched configs (4b, 5a): SURVEY.md 8(e) ----

def test_partition_by_cost_covers_every_instance_once():
    from paper_2502_03000_b200.datagen import batch_sizes
    from paper_2502_03000_b200.shard import partition_by_cost
    sizes = batch_sizes(262144)
    cost = sizes.astype(np.float64) ** 3
    for world in (1, 2, 3, 4, 8):
        parts = partition_by_cost(cost, world)
        assert parts[0][0] == 0 and parts[-1][1] == sizes.size
        assert all(parts[g][1] == parts[g + 1][0] for g in range(world - 1))
        shares = np.array([cost[lo:hi].sum() for lo, hi in parts]) / cost.sum()
        # balanced to within one n=128 instance of the ideal share
        assert np.max(np.abs(shares - 1.0 / world)) * cost.sum() <= 128.0 ** 3
    assert partition_by_cost([], 3) == [(0, 0)] * 3
    assert partition_by_cost(np.ones(5), 8)[-1][1] == 5


def test_class_ranges_are_contiguous_class_indices():
    from paper_2502_03000_b200.shard import class_ranges, partition_by_cost
    rng = np.random.default_rng(3)
    sizes = rng.choice([32, 64, 128], 1000)
    parts = partition_by_cost(sizes.astype(float) ** 3, 4)
    seen = {n: [] for n in (32, 64, 128)}
    for lo, hi in parts:
        for n, (first, count) in class_ranges(sizes, lo, hi, (32, 64, 128)).items():
            seen[n].append((first, count))
            # class index of each class-n instance in [lo, hi)
            idx = np.flatnonzero(sizes == n)
            mine = np.flatnonzero((idx >= lo) & (idx < hi))
            assert list(mine) == list(range(first, first + count))
    for n, lst in seen.items():
        assert lst[0][0] == 0 and sum(c for _, c in lst) == int((sizes == n).sum())


def _partition_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["WORLD_SIZE"], os.environ["RANK"] = str(world), str(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    wl = bench.Config5a()
    counts = torch.tensor([wl.ranges[n][1] for n in wl.SIZES] + [wl.hi - wl.lo], dtype=torch.int64)
    work = torch.tensor([float(wl._flops(wl.rank_counts()))], dtype=torch.float64)
    dist.all_reduce(counts)
    total_work = work.clone()
    dist.all_reduce(total_work)
    q.put((rank, wl.lo, wl.hi, counts.tolist(), float(work), float(total_work), wl.counts()))
    dist.destroy_process_group()


def test_bench_5a_partition_two_ranks_gloo():
    """bench.py's config-5a split at world size 2: every instance on exactly
    one rank, class counts add up to the batch, flops balanced."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partition_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    (r0, lo0, hi0, c0, w0, tw, full), (r1, lo1, hi1, c1, w1, _, _) = res
    assert (lo0, hi1) == (0, 262144) and hi0 == lo1
    assert c0 == c1 and c0[:3] == [full[32], full[64], full[128]] and c0[3] == 262144
    assert abs(w0 - w1) / tw < 1e-4
