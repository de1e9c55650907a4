"""Where the config-4b step's time goes: the solve_batched call vs its
kernels (device events) vs its host synchronisation."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200.batch import solve_batched, stack_fortran  # noqa: E402

n, bt = 64, 4096
rng = np.random.default_rng(1)
A = stack_fortran(rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None])
b = stack_fortran(rng.uniform(-1, 1, (bt, n, 1)))
for _ in range(5):
    solve_batched(A, b)
torch.cuda.synchronize()
K = 50
t = time.perf_counter()
for _ in range(K):
    solve_batched(A, b)
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / K * 1e6
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    solve_batched(A, b)
e1.record()
torch.cuda.synchronize()
print(f"solve_batched: wall {wall:.1f} us/step, events {e0.elapsed_time(e1) / K * 1e3:.1f} us/step")

from paper_2502_03000_b200 import _native as N  # noqa: E402
x = torch.empty((bt, 1, n), dtype=torch.float64, device="cuda").transpose(1, 2)
ci = torch.empty(2 * bt, dtype=torch.int32, device="cuda")
info = torch.empty(bt, dtype=torch.int32, device="cuda")
for name, fn in [("lu_solve_batched", lambda: N.call("lm_lu_solve_batched", 0, n, bt, A.data_ptr(), x.data_ptr(),
                                                          None, None, info.data_ptr())),
                 ("solve_batched_classified", lambda: N.call("lm_solve_batched_classified", 0, n, bt, A.data_ptr(),
                                                             x.data_ptr(), ci.data_ptr(), ci.data_ptr() + 4 * bt)),
                 ("x.copy_(b)", lambda: x.copy_(b))]:
    for _ in range(3):
        x.copy_(b)
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        x.copy_(b)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name}: {np.median(ts):.1f} us")
