"""Host-side cost of one evaluate() of a small expression (cProfile)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402

rng = np.random.default_rng(0)
A = lm.DenseMatrix(np.asfortranarray(rng.random((100, 100))))
B = lm.DenseMatrix(np.asfortranarray(rng.random((100, 100))))
for _ in range(200):
    lm.evaluate(0.4 * A + 0.6 * B)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(2000):
    lm.evaluate(0.4 * A + 0.6 * B)
torch.cuda.synchronize()
print(f"evaluate (1) 100^2: {(time.perf_counter() - t) / 2000 * 1e6:.1f} us per call")
cProfile.run("for _ in range(2000): lm.evaluate(0.4 * A + 0.6 * B)", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("tottime").print_stats(25)
