"""ctypes front end of the CPU oracle (oracle/lm_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this module.  The product package
``paper_2502_03000_b200`` must not (tests/test_boundary.py enforces it).

Each wrapper mirrors one ``lazymat._loops`` function
(/root/reference/pkg/src/lazymat/_loops.py) and accepts numpy float64
arrays of ANY stride, like the reference does (kernels.py:9-15): the
strides are passed through, so .T views, column/row windows and diagonal
views are read in place exactly as numba reads them.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liblm_oracle.so"

_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-std=c99", "-Wall"]


def build(force: bool = False) -> pathlib.Path:
    """Compile lm_oracle.c with FMA contraction disabled (bit-exact with
    numba, SURVEY.md finding 9)."""
    src = _HERE / "lm_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        _LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
        tmp = _LIB_PATH.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["gcc", *_CFLAGS, "-o", str(tmp), str(src), "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _View(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p), ("rows", ctypes.c_int64),
                ("cols", ctypes.c_int64), ("rs", ctypes.c_int64),
                ("cs", ctypes.c_int64)]


class _Vec(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p), ("n", ctypes.c_int64),
                ("stride", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
        V, Vp, I64p = _View, ctypes.POINTER(_View), ctypes.POINTER(ctypes.c_int64)
        d = ctypes.c_double
        sig = {
            "lmo_analyze": (None, [V, ctypes.c_int, I64p, I64p, ctypes.POINTER(ctypes.c_int)]),
            "lmo_fused": (None, [ctypes.c_int, ctypes.POINTER(d), Vp, V]),
            "lmo_program": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.POINTER(d), Vp, V]),
            "lmo_gemm": (None, [V, V, V]),
            "lmo_gemv": (None, [V, _Vec, _Vec, ctypes.c_int]),
            "lmo_syrk": (None, [V, V]),
            "lmo_diag_scale": (None, [_Vec, V, ctypes.c_int, V]),
            "lmo_diag_of_product": (None, [V, V, _Vec]),
            "lmo_trace_of_product": (d, [V, V]),
            "lmo_triple_diag_dot": (d, [_Vec, _Vec, _Vec]),
            "lmo_lu_factor": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
            "lmo_lu_solve": (None, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]),
            "lmo_pack_band": (None, [V, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]),
            "lmo_band_factor": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]),
            "lmo_band_solve": (None, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64]),
            "lmo_tri_solve": (ctypes.c_int, [V, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]),
            "lmo_transpose_copy": (None, [V, V]),
            "lmo_diag_materialise": (None, [_Vec, V]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _chk(a: np.ndarray) -> np.ndarray:
    if a.dtype != np.float64:
        raise TypeError(f"oracle works on float64, got {a.dtype}")
    return a


def view(a: np.ndarray) -> _View:
    _chk(a)
    if a.ndim != 2:
        raise ValueError("2-D view expected")
    s = a.strides
    return _View(a.ctypes.data, a.shape[0], a.shape[1], s[0] // 8, s[1] // 8)


def vec(a: np.ndarray) -> _Vec:
    _chk(a)
    if a.ndim != 1:
        raise ValueError("1-D vector expected")
    return _Vec(a.ctypes.data, a.shape[0], a.strides[0] // 8)


def _fortran_out(out):
    if not out.flags.writeable:
        raise ValueError("output must be writeable")
    return out


# ---- one wrapper per _loops function --------------------------------------

def analyze(a: np.ndarray, square: bool):
    """_loops.py:15-34 -> (lbw, ubw, sym)."""
    lbw, ubw, sym = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    lib().lmo_analyze(view(a), int(bool(square)), ctypes.byref(lbw), ctypes.byref(ubw), ctypes.byref(sym))
    return lbw.value, ubw.value, bool(sym.value)


def fused(coeffs, sources, out: np.ndarray) -> None:
    """_loops.py:37-84 (the fused_axpby_n family)."""
    n = len(coeffs)
    carr = (ctypes.c_double * n)(*[float(c) for c in coeffs])
    varr = (_View * n)(*[view(s) for s in sources])
    lib().lmo_fused(n, carr, varr, view(_fortran_out(out)))


def program(ops, args, consts, sources, out: np.ndarray) -> None:
    """Element-wise postfix program (extension op family)."""
    ops = np.ascontiguousarray(ops, dtype=np.int32)
    args = np.ascontiguousarray(args, dtype=np.int32)
    n = len(consts)
    carr = (ctypes.c_double * max(n, 1))(*[float(c) for c in consts])
    varr = (_View * max(len(sources), 1))(*[view(s) for s in sources])
    rc = lib().lmo_program(len(ops), ops.ctypes.data, args.ctypes.data, carr, varr,
                           view(_fortran_out(out)))
    if rc != 0:
        raise ValueError(f"malformed element-wise program (rc={rc})")


def gemm(a, b, out) -> None:
    """_loops.py:87-98."""
    lib().lmo_gemm(view(a), view(b), view(_fortran_out(out)))


def gemv(a, x, out, trans: bool = False) -> None:
    """_loops.py:101-121."""
    lib().lmo_gemv(view(a), vec(x), vec(_fortran_out(out)), int(bool(trans)))


def syrk(a, out) -> None:
    """_loops.py:124-141."""
    lib().lmo_syrk(view(a), view(_fortran_out(out)))


def diag_scale(d, b, side: str, out) -> None:
    """_loops.py:144-158."""
    lib().lmo_diag_scale(vec(d), view(b), int(side == "right"), view(_fortran_out(out)))


def diag_of_product(a, b, out_d) -> None:
    """_loops.py:161-176."""
    lib().lmo_diag_of_product(view(a), view(b), vec(_fortran_out(out_d)))


def trace_of_product(a, b) -> float:
    """_loops.py:179-188."""
    return float(lib().lmo_trace_of_product(view(a), view(b)))


def triple_diag_dot(a, d, c) -> float:
    """_loops.py:191-197."""
    return float(lib().lmo_triple_diag_dot(vec(a), vec(d), vec(c)))


def lu_factor(a):
    """_loops.py:200-236 on a fresh F-order copy -> (rc, lu, piv)."""
    lu = np.array(a, dtype=np.float64, order="F", copy=True)
    n = lu.shape[0]
    piv = np.zeros(n, dtype=np.int64)
    rc = lib().lmo_lu_factor(lu.ctypes.data, n, piv.ctypes.data)
    return rc, lu, piv


def lu_solve(lu, piv, x) -> None:
    """_loops.py:239-259; x (F-order, n x m) is overwritten."""
    assert lu.flags.f_contiguous and x.flags.f_contiguous
    piv = np.ascontiguousarray(piv, dtype=np.int64)
    n = lu.shape[0]
    m = x.shape[1]
    lib().lmo_lu_solve(lu.ctypes.data, n, piv.ctypes.data, x.ctypes.data, n, m)


def band_solve(a, x, kl: int, ku: int) -> int:
    """_loops.py:262-360 (pack, factor, substitute); returns rc."""
    n = a.shape[0]
    ldab = 2 * kl + ku + 1
    ab = np.zeros((ldab, n), order="F")
    piv = np.zeros(n, dtype=np.int64)
    L = lib()
    L.lmo_pack_band(view(a), ab.ctypes.data, ldab, kl, ku)
    rc = L.lmo_band_factor(ab.ctypes.data, ldab, n, piv.ctypes.data, kl, ku)
    if rc:
        return rc
    assert x.flags.f_contiguous
    L.lmo_band_solve(ab.ctypes.data, ldab, n, piv.ctypes.data, x.ctypes.data, n, x.shape[1], kl, ku)
    return 0


def tri_solve(a, x, upper: bool) -> int:
    """_loops.py:363-388; returns rc."""
    assert x.flags.f_contiguous
    return lib().lmo_tri_solve(view(a), x.ctypes.data, x.shape[0], x.shape[1], int(bool(upper)))


def transpose_copy(a, out) -> None:
    """_loops.py:391-396."""
    lib().lmo_transpose_copy(view(a), view(_fortran_out(out)))


def diag_materialise(d, out) -> None:
    """_loops.py:399-407."""
    lib().lmo_diag_materialise(vec(d), view(_fortran_out(out)))
