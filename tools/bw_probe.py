"""HBM calibration: torch copy vs our streaming kernels at several sizes
(CUDA-graph replays of 10 launches, CUDA events).  Prints GB/s per size."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_03000_b200 import kernels as K  # noqa: E402
from paper_2502_03000_b200.matrix import fortran_empty  # noqa: E402


def timed(fn, reps=10, iters=5):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(iters):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best * 1e-3


for n in (2048, 4096, 8192, 16384):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
    b = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
    o = fortran_empty(n, n)
    v = torch.rand(n, dtype=torch.float64, device="cuda")
    s = torch.empty(1, dtype=torch.float64, device="cuda")
    by = n * n * 8
    t_copy = timed(lambda: o.copy_(a))
    t_ds = timed(lambda: K.diag_scale(v, a, "left", o))
    t_dsr = timed(lambda: K.diag_scale(v, a, "right", o))
    t_tr = timed(lambda: K.trace_of_product(a, b, out=s))
    t_sum = timed(lambda: a.sum())
    print(f"n={n:6d} MB/op={by / 2**20:7.0f}  copy {2 * by / t_copy / 1e9:7.0f}  diag_scale L {2 * by / t_ds / 1e9:7.0f}"
          f"  R {2 * by / t_dsr / 1e9:7.0f}  trace {2 * by / t_tr / 1e9:7.0f}  torch.sum {by / t_sum / 1e9:7.0f} GB/s",
          flush=True)
    del a, b, o
    torch.cuda.empty_cache()
