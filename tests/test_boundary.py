"""The drop-in boundary, checked without a GPU.

* the C-ABI library is built for sm_100a, loads, and exports every entry
  point include/lm_b200.h declares (and _native binds);
* the product package never imports the oracle (parity would be void);
* with no CUDA device, evaluation fails loudly -- there is no CPU path;
* the extension planner output for BASELINE config 1 and the JIT source
  it generates.
"""

import ctypes
import pathlib
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_2502_03000_b200 as lm
from paper_2502_03000_b200 import _native
from paper_2502_03000_b200.build import build

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "lm_b200.h"
PKG = ROOT / "paper_2502_03000_b200"


@pytest.fixture(scope="module")
def libpath():
    return build()


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*\*?\s*(lm_\w+)\s*\(", text, re.M)))


def test_header_declares_the_bound_symbols():
    assert _declared() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(str(libpath))
    for name in _declared():
        assert hasattr(lib, name), name
    lib.lm_abi_version.restype = ctypes.c_int
    assert lib.lm_abi_version() == 1


def test_library_is_sm100a_sass(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", str(libpath)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(libpath)], capture_output=True, text=True).stdout
    assert "dgemm_dmma" in sass and "DMMA" in sass  # FP64 tensor-core path (mma.sync.m8n8k4.f64)


def test_product_never_imports_the_oracle():
    for f in PKG.rglob("*.py"):
        src = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
        assert "lm_oracle" not in src, f


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
def test_no_device_means_no_evaluation():
    a = lm.make_matrix(3, 3, "random", seed=1)
    with pytest.raises(lm.BackendUnavailableError):
        lm.evaluate(a + a)
    with pytest.raises(lm.BackendUnavailableError):
        lm.analyze_structure(a)


def test_config1_plan_is_one_fused_program():
    a, b, c = (lm.make_matrix(8, 8, "random", seed=s) for s in (1, 2, 3))
    plan = lm.rewrite(2 * a + b % c - a / (1 + abs(b)))
    assert plan.rule_log == ["R1"]
    assert [s.kernel for s in plan.steps] == ["fused_expr"]
    st = plan.steps[0]
    assert len(st.operands) == 3  # A and B are read once each
    assert st.params == ("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -", 2.0, 1.0)
    assert plan.slot_shapes == [(8, 8)]


def test_program_source_generation(libpath):
    lib = ctypes.CDLL(str(libpath))
    ops, args, *_ = lm.kernels.parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
    buf = ctypes.create_string_buffer(1 << 16)
    f = lib.lm_program_source
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                  ctypes.c_int, ctypes.c_char_p, ctypes.c_int64]
    assert f(0, 1, len(ops), ops.data_ptr(), args.data_ptr(), 2, 3, buf, len(buf)) == 0
    src = buf.value.decode()
    assert "__dmul_rn" in src and "__ddiv_rn" in src and "ld.global.nc" in src
    assert "fma" not in src.lower().replace("fmad", "")


def test_extension_semantics_pinned_to_naive():
    """The fused program of config 1 equals per-node (naive) IEEE
    evaluation bit for bit -- checked with the C oracle's program
    interpreter against numpy's per-node ufuncs."""
    from oracle import lm_oracle as O
    rng = np.random.default_rng(7)
    A, B, C = (np.asfortranarray(rng.uniform(-1, 1, (64, 48))) for _ in range(3))
    ops, args, _, _, _ = lm.kernels.parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
    out = np.zeros((64, 48), order="F")
    O.program(ops.numpy(), args.numpy(), [2.0, 1.0], [A, B, C], out)
    t1 = 2.0 * A
    t2 = B * C
    t3 = 1.0 * t1 + 1.0 * t2
    t6 = A / (1.0 + np.abs(B))
    naive = 1.0 * t3 + (-1.0) * t6
    assert np.array_equal(out.view(np.int64), naive.view(np.int64))


def test_capture_rejects_host_synchronising_plans():
    """Whole-plan CUDA-graph capture refuses plans with solves (they read
    the factorisation status / structure on the host) before touching a
    device."""
    from cases import CASES
    from paper_2502_03000_b200.errors import KernelContractError

    plan = lm.rewrite(CASES["r10_runtime_gen"](lm))
    assert "lu_solve" in [s.kernel for s in plan.steps]
    with pytest.raises(KernelContractError, match="not capturable"):
        lm.capture(plan)


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only check")
def test_capture_without_device_fails_loudly():
    from cases import CASES

    with pytest.raises(lm.BackendUnavailableError):
        lm.capture(CASES["r1_weighted_sum"](lm))
