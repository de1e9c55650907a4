"""Warm lu_factor runs of an n x n dominant matrix, the last one with the
LM_LU_TRACE timeline (stderr).  Prints the wall time of each run."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402
from paper_2502_03000_b200 import kernels as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
A0 = lm.DenseMatrix(rng.uniform(-1, 1, (n, n)) + n * np.eye(n))
for rep in range(4):
    A = A0.data.clone(memory_format=torch.contiguous_format) if False else A0.data.t().contiguous().t()
    torch.cuda.synchronize()
    if rep == 3:
        os.environ["LM_LU_TRACE"] = "1"
    t = time.perf_counter()
    K.lu_factor(A)
    th = time.perf_counter()
    torch.cuda.synchronize()
    print(f"lu_factor {n}: {(time.perf_counter() - t) * 1e3:.2f} ms (host issue {(th - t) * 1e3:.2f} ms)",
          file=sys.stderr)
