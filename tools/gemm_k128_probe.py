"""Throughput of the DMMA GEMM on the LU's trailing-update shapes (rank-128 / rank-32)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2502_03000_b200 import kernels as K  # noqa: E402
from paper_2502_03000_b200.matrix import fortran_empty  # noqa: E402


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (m, n, k) in [(8064, 7936, 128), (7000, 7000, 128), (4000, 4000, 128), (8064, 128, 128), (8160, 96, 32),
                  (2048, 2048, 2048), (16384, 16384, 128)]:
    a = fortran_empty(m, k)
    b = fortran_empty(k, n)
    c = fortran_empty(m, n)
    a.uniform_(-1, 1)
    b.uniform_(-1, 1)
    ms = t(lambda: K.gemm(a, b, c))
    print(f"gemm {m}x{k} * {k}x{n}: {ms * 1e3:8.1f} us  {2 * m * n * k / ms / 1e9:6.2f} TF/s")
