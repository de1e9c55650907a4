"""Per-phase cycle counts of the cluster LU panel kernel (lm_debug_lu_panel)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402
from paper_2502_03000_b200 import _native as N  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
A = lm.DenseMatrix(rng.uniform(-1, 1, (n, n)) + n * np.eye(n))
piv = torch.empty(n, dtype=torch.int64, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
clk = torch.zeros(4 * 32, dtype=torch.int64, device="cuda")
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    N.call("lm_debug_lu_panel", N.view(A.data), 0, 32, piv.data_ptr(), info.data_ptr(), clk.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    print("panel us", e0.elapsed_time(e1) * 1e3)
c = clk.cpu().numpy().reshape(32, 4)
d = np.diff(np.concatenate([c.reshape(-1), [c[-1, 3] + 0]]))
phases = np.stack([c[:, 1] - c[:, 0], c[:, 2] - c[:, 1], c[:, 3] - c[:, 2], np.r_[c[1:, 0] - c[:-1, 3], 0]], 1)
print("cycles per column by phase [argmax+publish, ctaCand+clusterSync, winner+dsmem, update]:")
print(phases[1:-1].mean(0), "total", phases[1:-1].sum(1).mean())
