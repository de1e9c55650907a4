"""Where an inverse(A)*b evaluation of a small matrix spends its time."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_03000_b200 as lm  # noqa: E402
from paper_2502_03000_b200 import kernels as K  # noqa: E402


def timeit(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e6


for n in (64, 100, 250, 500, 1000):
    rng = np.random.default_rng(n)
    A = lm.DenseMatrix(np.asfortranarray(rng.random((n, n)) + n * np.eye(n)))
    b = lm.DenseMatrix(np.asfortranarray(rng.random((n, 1))))
    x = torch.empty((n, 1), dtype=torch.float64, device="cuda")
    t_eval = timeit(lambda: lm.evaluate(lm.inverse(A) * b))
    t_rw = timeit(lambda: lm.rewrite(lm.inverse(A) * b))
    t_an = timeit(lambda: A.analyze_structure() if hasattr(A, "analyze_structure") else None)
    t_fac = timeit(lambda: K.lu_factor(A.data))
    t_sol = timeit(lambda: K.lu_solve_into(A.data, x.copy_(b.data)))
    print(f"n={n}: evaluate {t_eval:.0f} us | rewrite {t_rw:.0f} | analyze {t_an:.0f} | lu_factor {t_fac:.0f} | "
          f"factor+solve {t_sol:.0f}")
