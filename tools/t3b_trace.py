"""Phase times of the skinny GEMM kernels on config 3b's shapes (LM_SKINNY_TRACE=1)."""
import os, sys
os.environ["LM_SKINNY_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_03000_b200 as lm

rng = np.random.default_rng(3)
X = lm.DenseMatrix(rng.uniform(-1, 1, (8000, 100)))
Y = lm.DenseMatrix(rng.uniform(-1, 1, (100, 8000)))
Z = lm.DenseMatrix(rng.uniform(-1, 1, (8000, 100)))
for _ in range(4):
    out = lm.evaluate(X * Y * Z)
    torch.cuda.synchronize()
