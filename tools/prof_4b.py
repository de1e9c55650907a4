"""Device time of one lm_lu_solve_batched launch on config 4b (4096 x 64^2)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200 import _native as N  # noqa: E402
from paper_2502_03000_b200.batch import stack_fortran  # noqa: E402
n, bt = 64, int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(1000003 * 42 + 101 * 4 + 7)
A = stack_fortran(rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None])
b = stack_fortran(rng.uniform(-1, 1, (bt, n, 1)))
x = torch.empty((bt, 1, n), dtype=torch.float64, device="cuda").transpose(1, 2)
info = torch.empty(bt, dtype=torch.int32, device="cuda")


def solve():
    x.copy_(b)
    N.call("lm_lu_solve_batched", 0, n, bt, A.data_ptr(), x.data_ptr(), None, None, info.data_ptr())


solve()
torch.cuda.synchronize()
ts = []
for _ in range(9):
    x.copy_(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    N.call("lm_lu_solve_batched", 0, n, bt, A.data_ptr(), x.data_ptr(), None, None, info.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"4b lu_solve_batched n={n} batch={bt}: {ms * 1e3:.1f} us  "
      f"{bt * (2 * n ** 3 // 3 + 2 * n * n) / ms / 1e9:.2f} TF/s  {bt * (n * n * 8 + 16 * n) / ms / 1e6:.0f} GB/s")
