"""Per-phase cycle counts of the cluster LU panel kernel (lm_debug_lu_panel):
clock64 marks of CTA 0 / thread 0 per column:
 0 iteration start, 1 after cluster wait, 2 after winner/U copy, 3 after
 swap + multipliers + next-column update, 4 after warp argmax/publish,
 5 after __syncthreads, 6 after pushes + arrive, 7 after the rest of the update."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402
from paper_2502_03000_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
A0 = lm.DenseMatrix(rng.uniform(-1, 1, (n, n)) + n * np.eye(n))
piv = torch.empty(n, dtype=torch.int64, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
clk = torch.zeros(8 * 32 + 8, dtype=torch.int64, device="cuda")
for rep in range(3):
    A = A0.data.t().contiguous().t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    N.call("lm_debug_lu_panel", N.view(A), 0, 32, piv.data_ptr(), info.data_ptr(), clk.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    print("panel us", e0.elapsed_time(e1) * 1e3)
allc = clk.cpu().numpy().astype(np.float64)
c = allc[:256].reshape(32, 8)
t = allc[256:260]
print("kernel phases (cycles): load+cluster sync %.0f, column loop %.0f, write-back %.0f" % (t[1] - t[0], t[2] - t[1], t[3] - t[2]))
names = ["wait", "winner", "swap+col", "argmax", "syncthr", "push+arrive", "rest upd", "->next"]
d = np.stack([c[:, 1] - c[:, 0], c[:, 2] - c[:, 1], c[:, 3] - c[:, 2], c[:, 4] - c[:, 3], c[:, 5] - c[:, 4],
              c[:, 6] - c[:, 5], c[:, 7] - c[:, 6], np.r_[c[1:, 0] - c[:-1, 7], 0]], 1)
m = d[1:-1].mean(0)
print("cycles per column:", ", ".join(f"{k} {v:.0f}" for k, v in zip(names, m)), "| total", m.sum())
