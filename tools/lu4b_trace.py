"""Per-warp phase timeline of the pivot-free batched LU (config 4b): run
with LM_4B_TRACE=1; lane 0 of each warp records clock64() at the phase
boundaries (csrc/lu_batched.cu, LU4B_MARK): slots 0 start, 1+3kb block
start, 2+3kb after B1, 3+3kb after B2, 25 back sweep start, 26 end,
27+kb end of (c) (kb < 4), 31 SM id.   Usage: lu4b_trace.py [batch]"""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200 import _native as N  # noqa: E402
from paper_2502_03000_b200.batch import stack_fortran  # noqa: E402
import ctypes  # noqa: E402
import cuda.bindings.runtime as rt  # noqa: E402

n, bt = 64, int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(7)
A = stack_fortran(rng.uniform(-1, 1, (bt, n, n)) + n * np.eye(n)[None])
b = stack_fortran(rng.uniform(-1, 1, (bt, n, 1)))
x = torch.empty((bt, 1, n), dtype=torch.float64, device="cuda").transpose(1, 2)
info = torch.empty(bt, dtype=torch.int32, device="cuda")
lib = N.load_library()
lib.lm_debug_lu4b_trace.restype = ctypes.c_void_p
for _ in range(3):
    x.copy_(b)
    N.call("lm_lu_solve_batched", 0, n, bt, A.data_ptr(), x.data_ptr(), None, None, info.data_ptr())
torch.cuda.synchronize()
ptr = lib.lm_debug_lu4b_trace()
host = np.zeros(64 * bt, dtype=np.int64)
rt.cudaMemcpy(host.ctypes.data, ptr, host.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
tr = host.reshape(bt, 2, 32)
t0 = tr[:, :, 0].min(axis=1)
rel = tr[:, :, :31] - t0[:, None, None]
print(f"batch {bt}: CTA duration mean {rel[:, :, 26].max(axis=1).mean():.0f} cycles")
for w in range(2):
    print(f"warp {w}:")
    for kb in range(8):
        st = rel[:, w, 1 + 3 * kb].mean()
        b1 = rel[:, w, 2 + 3 * kb].mean()
        b2 = rel[:, w, 3 + 3 * kb].mean()
        nx = rel[:, w, 1 + 3 * (kb + 1)].mean() if kb < 7 else rel[:, w, 25].mean()
        c = f" (c) {rel[:, w, 27 + kb].mean() - b1:6.0f}" if kb < 4 else ""
        print(f"  block {kb}: start {st:7.0f}  ->B1 {b1 - st:6.0f}  B1->B2 {b2 - b1:6.0f}{c}  (d) {nx - b2:6.0f}")
    print(f"  back sweep {rel[:, w, 26].mean() - rel[:, w, 25].mean():.0f}")
