import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200 import _native as N
from paper_2502_03000_b200.batch import stack_fortran
n, bt = 64, 4096
rng = np.random.default_rng(5)
A = stack_fortran(rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None])
b = stack_fortran(rng.uniform(-1, 1, (bt, n, 1)))
x = torch.empty((bt, 1, n), dtype=torch.float64, device="cuda").transpose(1, 2)
x.copy_(b)
info = torch.zeros(bt, dtype=torch.int32, device="cuda")
N.call("lm_lu_solve_batched", 0, n, bt, A.data_ptr(), x.data_ptr(), None, None, info.data_ptr())
torch.cuda.synchronize()
i = info.cpu().numpy()
print("redo count", (i == -1).sum(), "of", bt, "other nonzero", ((i != 0) & (i != -1)).sum())
