"""Time the pieces of the 8192 LU solve (config 4a) with CUDA events."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402
from paper_2502_03000_b200 import kernels as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
a = rng.uniform(-1, 1, (n, n)) + n * np.eye(n)
A = lm.DenseMatrix(a)
B = lm.DenseMatrix(rng.uniform(-1, 1, (n, 64)))


def ev(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


print("lu_factor", ev(lambda: K.lu_factor(A.data)))
lu, piv = K.lu_factor(A.data)
x = B.data.clone()
from paper_2502_03000_b200 import _native as N  # noqa: E402
print("lu_solve", ev(lambda: N.call("lm_lu_solve", 0, N.view(lu.data), piv.data_ptr(), N.view(x))))
print("analyze", ev(lambda: lm.analyze_structure(A)))
print("evaluate", ev(lambda: lm.evaluate(lm.inverse(A) * B)))
