"""The n = 128 batched-expression kernels have A/B baselines behind
environment switches (read once per process): TMA-fed vs cp.async-fed rings,
tcgen05 vs legacy mma.sync TF32, the streaming vs the two-CTA cluster f64
kernel.  Each variant runs in a subprocess on the same seeded batch and must
agree with the oracle-checked default within the north-star tolerance."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]
SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2502_03000_b200.batch import atb_schur_trace, stack_fortran
from paper_2502_03000_b200 import _native
dt = torch.float64 if sys.argv[2] == "f64" else torch.float32
import os
rng = np.random.default_rng(11)
n = int(os.environ.get("LM_5A_N", "128"))
bt = 400 if n == 128 else 401
ops = [rng.uniform(-1, 1, (bt, n, n)) for _ in range(4)]
E, s = atb_schur_trace(*(stack_fortran(o, dtype=dt) for o in ops))
variant = _native.last_variant()
idx = [0, 1, 147, 148, 296, 299, 399]
print(json.dumps({"E": E[idx].double().cpu().numpy().ravel()[::97].tolist(), "s": s[idx].double().cpu().tolist(),
                  "variant": variant}))
"""


def run(env_extra, dtype):
    env = dict(os.environ)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), dtype], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def close(a, b, tol):
    import numpy as np
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b)) <= tol * max(np.max(np.abs(b)), 1e-30)


@pytest.mark.parametrize("variant,kernel", [({"LM_5A_TM": "1"}, "stream_tm"), ({"LM_5A_WS": "0"}, "stream_tma"),
                                            ({"LM_5A_MW": "8"}, "stream_ws8"),
                                            ({"LM_5A_TMA": "0"}, "stream"), ({"LM_5A_STREAM": "0"}, "half")])
def test_f64_variants_agree(variant, kernel):
    ref = run({}, "f64")
    assert ref["variant"] == "stream_ws"
    got = run(variant, "f64")
    assert got["variant"] == kernel  # the switch selected the kernel it names
    assert close(got["E"], ref["E"], 1e-12) and close(got["s"], ref["s"], 1e-12)


@pytest.mark.parametrize("variant,kernel", [({"LM_5A_TC05": "1"}, "tc05"), ({"LM_5A_TC05": "0"}, "stream_f32"),
                                            ({"LM_5A_TF32": "0"}, "tc_f32_128")])
def test_f32_variants_agree(variant, kernel):
    ref = run({}, "f32")
    assert ref["variant"] == "tc05t"
    got = run(variant, "f32")
    assert got["variant"] == kernel
    assert close(got["E"], ref["E"], 1e-5) and close(got["s"], ref["s"], 1e-5)


@pytest.mark.parametrize("n", [32, 64])
def test_f32_grouped_small_sizes_agree(n):
    """n = 64 in pairs (default) and n = 32 in groups of four (LM_5A_TC05Q=1)
    per 128 x 128 tcgen05 tile vs the FFMA kernel (LM_5A_TC05P=0), 401
    instances (a partial last group)."""
    ref = run({"LM_5A_TC05P": "0", "LM_5A_N": str(n)}, "f32")
    got = run({"LM_5A_TC05Q": "1", "LM_5A_N": str(n)}, "f32")
    assert ref["variant"] == f"tc_f32_{n}"
    assert got["variant"] == f"tc05p{n}"  # the grouped tcgen05 kernel really ran
    assert close(got["E"], ref["E"], 1e-5) and close(got["s"], ref["s"], 1e-5)


LU_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2502_03000_b200.batch import solve_batched, stack_fortran
from paper_2502_03000_b200 import _native
rng = np.random.default_rng(21)
n, bt = 64, 300
A = rng.uniform(-1, 1, (bt, n, n))
A[::2] += n * np.eye(n)[None]          # dominant half: pivot-free path; the rest pivots
b = rng.uniform(-1, 1, (bt, n, 1))
x = solve_batched(stack_fortran(A), stack_fortran(b), check=False).x
variant = _native.last_variant()
print(json.dumps({"x": x.cpu().numpy().view(np.int64).ravel()[::7].tolist(), "variant": variant}))
"""


def run_lu(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", LU_SCRIPT, str(ROOT)], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("variant,kernel", [({"LM_BATCHED_LU": "shift"}, "shift64"),
                                            ({"LM_BATCHED_LU": "wave"}, "wave64"),
                                            ({"LM_BATCHED_LU": "rows"}, "rows")])
def test_batched_lu_variants_bitwise(variant, kernel):
    """Config 4b's kernels: the blocked pivot-free fast path (default)
    against the unblocked pivot-free wavefront kernel, the round-1 pivoting
    kernel on every system and the unrolled kernel, on a batch where half
    the systems pivot: bit-identical solutions."""
    ref = run_lu({})
    assert ref["variant"] == "nopiv64"
    got = run_lu(variant)
    assert got["variant"] == kernel
    assert got["x"] == ref["x"]


GEMM_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2502_03000_b200 as lm
from paper_2502_03000_b200 import _native
rng = np.random.default_rng(31)
X = lm.DenseMatrix(rng.uniform(-1, 1, (300, 78)))
Y = lm.DenseMatrix(rng.uniform(-1, 1, (78, 2050)))
A = lm.DenseMatrix(rng.uniform(-1, 1, (1000, 130)))
P = lm.evaluate(X * Y).to_numpy()
v1 = _native.last_variant()
S = lm.evaluate(A.t() * A).to_numpy()
print(json.dumps({"P": P.view(np.int64).ravel()[::97].tolist(), "S": S.view(np.int64).ravel()[::13].tolist(),
                  "variant": v1, "variant_syrk": _native.last_variant()}))
"""


def test_gemm_tma_and_cp_async_kernels_bitwise():
    """The TMA-fed GEMM/SYRK kernel (default) and the cp.async kernel
    (LM_GEMM_TMA=0) run the same tiles in the same K order: bit-identical
    products, edge tiles (300 x 2050, K = 78 / 1000) included."""
    def run_g(env_extra):
        env = dict(os.environ)
        env.update(env_extra)
        out = subprocess.run([sys.executable, "-c", GEMM_SCRIPT, str(ROOT)], env=env, capture_output=True, text=True,
                             timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        return json.loads(out.stdout.strip().splitlines()[-1])
    ref = run_g({})
    assert ref["variant"] == "gemm_tma" and ref["variant_syrk"] == "gemm_tma"
    got = run_g({"LM_GEMM_TMA": "0"})
    assert got["variant"] == "gemm_cp" and got["variant_syrk"] == "gemm_cp"
    assert got["P"] == ref["P"] and got["S"] == ref["S"]


def test_gemm_wide_tile_kernel_bitwise():
    """The opt-in 64 x 128-tile TMA kernel (LM_GEMM_WIDE=1) on a product
    100 columns wide agrees with the default kernel normwise to 1e-12 (the
    split-K grouping follows the tile count, so the sums may associate
    differently)."""
    script = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2502_03000_b200 as lm
from paper_2502_03000_b200 import _native
rng = np.random.default_rng(32)
X = lm.DenseMatrix(rng.uniform(-1, 1, (1000, 300)))
T = lm.DenseMatrix(rng.uniform(-1, 1, (300, 100)))
P = lm.evaluate(X * T).to_numpy()
print(json.dumps({"P": P.ravel()[::31].tolist(), "variant": _native.last_variant()}))
"""
    outs = []
    for env_extra in ({}, {"LM_GEMM_WIDE": "1"}):
        env = dict(os.environ)
        env.update(env_extra)
        out = subprocess.run([sys.executable, "-c", script, str(ROOT)], env=env, capture_output=True, text=True,
                             timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    assert outs[0]["variant"] == "gemm_tma" and outs[1]["variant"] == "gemm_tma_wide"
    assert close(outs[1]["P"], outs[0]["P"], 1e-12)


def test_gemv_row_owner_and_split_k_kernels_agree():
    """The row-owner GEMV (default for column-major f64, no split-K finish)
    and the split-K kernel (LM_GEMV_ROWS=0) agree normwise to 1e-12 on a
    4096 x 4096 matrix-vector product and on a ragged 1000 x 777 one."""
    script = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2502_03000_b200 as lm
from paper_2502_03000_b200 import _native
rng = np.random.default_rng(33)
out = {}
for p, q in ((4096, 4096), (1000, 777)):
    M = lm.DenseMatrix(rng.uniform(-1, 1, (p, q)))
    v = lm.DenseMatrix(rng.uniform(-1, 1, (q, 1)))
    out[f"{p}x{q}"] = lm.evaluate(M * v).to_numpy().ravel()[::7].tolist()
    out[f"v{p}"] = _native.last_variant()
print(json.dumps(out))
"""
    outs = []
    for env_extra in ({}, {"LM_GEMV_ROWS": "0"}):
        env = dict(os.environ)
        env.update(env_extra)
        out = subprocess.run([sys.executable, "-c", script, str(ROOT)], env=env, capture_output=True, text=True,
                             timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    assert outs[0]["v4096"] == "gemv_rows" and outs[0]["v1000"] == "gemv_rows"
    assert outs[1]["v4096"] != "gemv_rows"
    for key in ("4096x4096", "1000x777"):
        assert close(outs[0][key], outs[1][key], 1e-12)
