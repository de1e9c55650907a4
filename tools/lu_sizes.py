"""lu_factor time of n x n dominant matrices (tensor mode, pivot-free path) for several n:
how much of config 4a's 8192 factorisation is the latency-bound tail."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402
from paper_2502_03000_b200 import kernels as K  # noqa: E402
for n in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096, 8192]:
    rng = np.random.default_rng(0)
    A = lm.DenseMatrix(rng.uniform(-1, 1, (n, n)) + n * np.eye(n))
    ts = []
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lu, piv = K.lu_factor(A.data, mode="tensor")
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        del lu, piv
    print(f"n={n}: lu_factor {min(ts[1:]):.3f} ms ({n // 128} outer blocks, {min(ts[1:]) * 1e3 / (n / 128):.0f} us per block, "
          f"{2 * n ** 3 / 3 / (min(ts[1:]) * 1e-3) / 1e12:.2f} TFLOP/s)")
