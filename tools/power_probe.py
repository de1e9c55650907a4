"""Clock / power / throttle reasons while one kernel variant runs back to back
(is the n = 128 f64 batched kernel power-capped?)."""
import statistics
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200.batch import atb_schur_trace, empty_batch  # noqa: E402
from paper_2502_03000_b200.datagen import fill_batch_class  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
bt = int(sys.argv[2]) if len(sys.argv) > 2 else 40000
ops = [fill_batch_class(empty_batch(bt, n, n), k, n, 0) for k in range(4)]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sample():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.01)


atb_schur_trace(*ops)
torch.cuda.synchronize()
t = threading.Thread(target=sample)
t.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 0
t0 = time.time()
while time.time() - t0 < 3.0:
    for _ in range(20):
        atb_schur_trace(*ops)
    reps += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
stop.set()
t.join()
ms = e0.elapsed_time(e1) / reps
clk = [c for c, p, r in samples[5:]]
pw = [p for c, p, r in samples[5:]]
reasons = 0
for c, p, r in samples[5:]:
    reasons |= r
print(f"n={n} {ms:.3f} ms/launch  sm_mhz median {statistics.median(clk)} min {min(clk)} max {max(clk)}  "
      f"power median {statistics.median(pw):.0f} W max {max(pw):.0f} W  reasons 0x{reasons:x}")
