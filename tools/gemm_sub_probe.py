"""The blocked LU's trailing update C -= L21 U12 (lm_debug_gemm_sub) alone, on config 4a's
shapes and operand layout (blocks of one 8192 x 8192 F-order matrix): its rate without the
panel chain next to it."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2502_03000_b200 import _native as N  # noqa: E402
from paper_2502_03000_b200.matrix import fortran_empty  # noqa: E402

n = 8192
A = fortran_empty(n, n)
A.uniform_(-1, 1)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


total = 0.0
for J0 in range(0, n - 128, 128):
    J1, J2 = J0 + 128, min(J0 + 256, n)
    if J2 >= n:
        break
    a, b, c = A[J1:, J0:J1], A[J0:J1, J2:], A[J1:, J2:]
    ms = t(lambda: N.call("lm_debug_gemm_sub", N.view(a), N.view(b), N.view(c)), reps=3)
    total += ms
    if J0 % 1024 == 0:
        m, nn = a.shape[0], b.shape[1]
        print(f"J0={J0}: {m}x128 * 128x{nn}: {ms * 1e3:7.1f} us  {2 * m * nn * 128 / ms / 1e9:6.2f} TF/s")
print(f"all trailing updates of the 8192 factorisation, alone: {total:.2f} ms")
