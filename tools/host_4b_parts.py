"""Host-side cost of the parts of solve_batched (config 4b) between two
device synchronisations: the GPU idles for the pre-launch part."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200 import _native as N  # noqa: E402
from paper_2502_03000_b200.batch import _check_batch, _pinned_i32, stack_fortran  # noqa: E402

n, bt = 64, 4096
rng = np.random.default_rng(1)
A = stack_fortran(rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None])
b = stack_fortran(rng.uniform(-1, 1, (bt, n, 1)))
T = {k: [] for k in ("check", "alloc+copy", "ci+launch", "readback", "post")}
for rep in range(60):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _check_batch(A, "A")
    _check_batch(b, "b")
    t1 = time.perf_counter()
    x = torch.empty((bt, 1, n), dtype=A.dtype, device=A.device).transpose(1, 2)
    x.as_strided((x.numel(),), (1,)).copy_(b.as_strided((b.numel(),), (1,), b.storage_offset()))
    t2 = time.perf_counter()
    ci = torch.empty(2 * bt, dtype=torch.int32, device=A.device)
    N.call("lm_solve_batched_classified", N.dtype_code(A), n, bt, A.data_ptr(), x.data_ptr(), ci.data_ptr(),
           ci.data_ptr() + 4 * bt)
    t3 = time.perf_counter()
    host_t = _pinned_i32(2 * bt)
    host_t.copy_(ci, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    t4 = time.perf_counter()
    host = host_t.numpy()
    ok = not host.any()
    t5 = time.perf_counter()
    if rep >= 10:
        for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
            T[k].append(v * 1e6)
print({k: round(float(np.median(v)), 1) for k, v in T.items()})
