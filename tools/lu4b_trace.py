"""Phase timeline of the pivot-free batched LU (config 4b): run with
LM_4B_TRACE=1; thread 63 of every CTA records clock64() at the phase
boundaries (csrc/lu_batched.cu, LU4B_MARK)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200 import _native as N  # noqa: E402
from paper_2502_03000_b200.batch import stack_fortran  # noqa: E402

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
host = np.zeros(32 * bt, dtype=np.int64)
torch.cuda.synchronize()
import cuda.bindings.runtime as rt  # noqa: E402
rt.cudaMemcpy(host.ctypes.data, ptr, host.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
if False: (
                                       0)
tr = host.reshape(bt, 32)
t0 = tr[:, 0]
rel = tr[:, :27] - t0[:, None]
dur = rel[:, 26]
print(f"CTA duration: mean {dur.mean():.0f} cycles, median {np.median(dur):.0f}, min {dur.min()}, max {dur.max()}")
ph = {"a": [], "bc": [], "d": []}
for kb in range(8):
    a = rel[:, 2 + 3 * kb] - rel[:, 1 + 3 * kb]
    bc = rel[:, 3 + 3 * kb] - rel[:, 2 + 3 * kb]
    d = (rel[:, 1 + 3 * (kb + 1)] if kb < 7 else rel[:, 25]) - rel[:, 3 + 3 * kb]
    print(f"block {kb}: (a)+B1 {a.mean():7.0f}  (b,c)+B2 {bc.mean():7.0f}  (d) {d.mean():7.0f}")
print(f"prologue {rel[:, 1].mean():.0f}  back sweep {(rel[:, 26] - rel[:, 25]).mean():.0f}")
sm = tr[:, 30]
print("CTAs per SM:", np.bincount(sm.astype(int)).min(), np.bincount(sm.astype(int)).max())
