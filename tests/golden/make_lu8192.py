"""Golden digests of the config-4a solve at full size (n = 8192, 64 RHS).

Runs the C oracle (oracle/lm_oracle.c: lazymat/_loops.py:200-259 restated,
pinned bitwise to the reference by tests/test_oracle_golden.py) once on the
bench's seeded inputs (bench.py Config4a: A = U(-1,1) + 8192*I with seed
1000003*42 + 101*4 + 0, b = U(-1,1) with seed ... + 1) and records SHA-256
digests of the LU factors, the pivots and the solution, plus a few sampled
values.  The factorisation takes several minutes on one core, too long for
the GPU test budget, so tests/test_gpu_fullsize.py compares the device's
exact-order LU against these digests instead of re-running the oracle.

    python tests/golden/make_lu8192.py   # writes tests/golden/lu8192.json
"""
import hashlib
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import lm_oracle as O  # noqa: E402

N, K = 8192, 64


def inputs():
    a = np.asfortranarray(np.random.default_rng(1000003 * 42 + 101 * 4 + 0).uniform(-1.0, 1.0, (N, N)))
    a[np.diag_indices(N)] += N
    b = np.asfortranarray(np.random.default_rng(1000003 * 42 + 101 * 4 + 1).uniform(-1.0, 1.0, (N, K)))
    return a, b


def digest(x) -> str:
    return hashlib.sha256(np.asfortranarray(x).tobytes(order="F")).hexdigest()


def main():
    a, b = inputs()
    t0 = time.time()
    rc, lu, piv = O.lu_factor(a)
    x = np.array(b, order="F")
    O.lu_solve(lu, piv, x)
    out = {"n": N, "nrhs": K, "rc": int(rc), "lu_sha256": digest(lu), "piv_sha256": digest(piv.astype(np.int64)),
           "x_sha256": digest(x), "piv_is_identity": bool(np.array_equal(piv, np.arange(N))),
           "x_samples": {f"{i},{j}": float(x[i, j]) for i, j in [(0, 0), (1, 5), (4095, 17), (8191, 63)]},
           "oracle_seconds": round(time.time() - t0, 1)}
    (ROOT / "tests" / "golden" / "lu8192.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
