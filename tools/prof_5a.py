"""One profiled launch of a config-5a size class (ncu target)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200.batch import atb_schur_trace, empty_batch
from paper_2502_03000_b200.datagen import fill_batch_class
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
bt = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
dt = torch.float64 if (len(sys.argv) <= 3 or sys.argv[3] == "f64") else torch.float32
ops = [fill_batch_class(empty_batch(bt, n, n, dt), k, n, 0) for k in range(4)]
for _ in range(2):
    E, s = atb_schur_trace(*ops)
torch.cuda.synchronize()
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    E, s = atb_schur_trace(*ops)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
w = 8 if dt == torch.float64 else 4
print(f"n={n} bt={bt} {ms:.3f} ms  {bt * 5 * n * n * w / ms / 1e6:.0f} GB/s  {bt * 2 * n ** 3 / ms / 1e9:.2f} TF/s")
