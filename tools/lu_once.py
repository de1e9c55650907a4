"""One lu_factor of an n x n dominant matrix (for ncu launch lists)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402
from paper_2502_03000_b200 import kernels as K  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
A = lm.DenseMatrix(rng.uniform(-1, 1, (n, n)) + n * np.eye(n))
K.lu_factor(A.data)
torch.cuda.synchronize()
