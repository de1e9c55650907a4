"""Time single lm_gemm calls (CUDA events, warm) for given shapes.
usage: python tools/gemm_probe.py M K N [M K N ...]"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch

from paper_2502_03000_b200 import kernels as K
from paper_2502_03000_b200.matrix import fortran_empty


def main():
    dims = [int(x) for x in sys.argv[1:]]
    for i in range(0, len(dims), 3):
        m, k, n = dims[i:i + 3]
        a = torch.rand((k, m), dtype=torch.float64, device="cuda").t()  # F-order m x k
        b = torch.rand((n, k), dtype=torch.float64, device="cuda").t()
        out = fortran_empty(m, n, device="cuda")
        for _ in range(5):
            K.gemm(a, b, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record()
        for _ in range(reps):
            K.gemm(a, b, out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        print(f"gemm {m}x{k}x{n}: {us:.2f} us  {2 * m * n * k / us / 1e6:.2f} TF/s", flush=True)


if __name__ == "__main__":
    main()
