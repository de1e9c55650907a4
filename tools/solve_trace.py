import os, sys, numpy as np, torch
os.environ["LM_SOLVE_TRACE"] = "1"
sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm
from paper_2502_03000_b200 import kernels as K
n, k = 8192, 64
rng = np.random.default_rng(0)
A = lm.DenseMatrix(rng.uniform(-1, 1, (n, n)) + n * np.eye(n))
b = torch.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (n, k)))).cuda()
lu, piv = K.lu_factor(A.data)
from paper_2502_03000_b200 import _native as N
from paper_2502_03000_b200.matrix import fortran_empty
x = fortran_empty(n, k); 
for rep in range(3):
    x.copy_(b)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); N.call("lm_lu_solve", 0, N.view(lu.data), piv.data_ptr(), N.view(x)); e1.record(); torch.cuda.synchronize()
    print("solve ms", e0.elapsed_time(e1), file=sys.stderr)
