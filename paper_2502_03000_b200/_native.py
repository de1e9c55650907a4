"""ctypes binding of the sm_100a C-ABI library (include/lm_b200.h).

This is the drop-in seam: it takes the place of the reference's numba
loop module (lazymat/_loops.py:15-407).  Operands are torch CUDA tensors
of any stride -- torch is used only as the device-memory owner and for
the current stream; all arithmetic happens in our kernels.  A call that
fails in the library raises BackendError with the library's message.

There is deliberately no CPU fallback: without a CUDA device (or
without the built library) every compute entry point raises
BackendUnavailableError.
"""

from __future__ import annotations

import ctypes
import pathlib
import threading

import torch

from .errors import BackendError, BackendUnavailableError

LIB_PATH = pathlib.Path(__file__).resolve().parent / "_lib" / "liblm_b200.so"

F64, F32 = 0, 1
LU_MODES = {"auto": 0, "exact": 1, "tensor": 2}  # lm_lu_factor_mode (include/lm_b200.h)

# Every symbol include/lm_b200.h declares (checked by tests/test_boundary.py).
EXPORTS = (
    "lm_abi_version", "lm_last_error", "lm_launch_count", "lm_last_variant",
    "lm_fused_axpby", "lm_fused_program", "lm_program_source", "lm_copy", "lm_vec_sum",
    "lm_gemm", "lm_gemm_chain", "lm_gemv", "lm_syrk",
    "lm_diag_scale", "lm_diag_of_product", "lm_trace_of_product", "lm_triple_diag_dot",
    "lm_analyze", "lm_lu_factor", "lm_lu_factor_mode", "lm_lu_factor_from", "lm_lu_solve", "lm_lu_solve_mode", "lm_band_solve", "lm_tri_solve",
    "lm_transpose_copy", "lm_diag_materialise", "lm_set_identity",
    "lm_lu_solve_batched", "lm_solve_batched_classified", "lm_solve_batched_classified_from", "lm_analyze_batched", "lm_expr_atb_schur_trace_batched", "lm_fill_uniform",
    "lm_fill_pcg64", "lm_nccl_load", "lm_nccl_unique_id", "lm_nccl_init_rank", "lm_nccl_init_all",
    "lm_allreduce_sum", "lm_allreduce_sum_f64", "lm_nccl_destroy",
    "lm_debug_lu_panel", "lm_debug_gemm_sub",
)


class View(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("rs", ctypes.c_int64), ("cs", ctypes.c_int64)]


class Vec(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("n", ctypes.c_int64), ("stride", ctypes.c_int64)]


_i, _i64, _p, _d = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
_SIGS = {
    "lm_abi_version": (_i, []),
    "lm_last_error": (ctypes.c_char_p, []),
    "lm_launch_count": (_i64, []),
    "lm_last_variant": (ctypes.c_char_p, []),
    "lm_fused_axpby": (_i, [_i, _i, ctypes.POINTER(_d), ctypes.POINTER(View), View, _p]),
    "lm_fused_program": (_i, [_i, _i, _p, _p, _i, ctypes.POINTER(_d), _i, ctypes.POINTER(View), View, _p]),
    "lm_program_source": (_i, [_i, _i, _i, _p, _p, _i, _i, ctypes.c_char_p, _i64]),
    "lm_copy": (_i, [_i, View, View, _p]),
    "lm_vec_sum": (_i, [_i, Vec, _p, _p]),
    "lm_gemm": (_i, [_i, View, View, View, _p]),
    "lm_gemm_chain": (_i, [_i, View, View, View, View, View, _p]),
    "lm_gemv": (_i, [_i, View, Vec, Vec, _i, _p]),
    "lm_syrk": (_i, [_i, View, View, _p]),
    "lm_diag_scale": (_i, [_i, Vec, View, _i, View, _p]),
    "lm_diag_of_product": (_i, [_i, View, View, Vec, _p]),
    "lm_trace_of_product": (_i, [_i, View, View, _p, _p]),
    "lm_triple_diag_dot": (_i, [_i, Vec, Vec, Vec, _p, _p]),
    "lm_analyze": (_i, [_i, View, _i, _p, _p]),
    "lm_lu_factor": (_i, [_i, View, _p, _p, _p]),
    "lm_lu_factor_mode": (_i, [_i, View, _p, _p, _i, _p]),
    "lm_lu_factor_from": (_i, [_i, View, View, _p, _p, _i, _p]),
    "lm_lu_solve": (_i, [_i, View, _p, View, _p]),
    "lm_lu_solve_mode": (_i, [_i, View, _p, View, _i, _p]),
    "lm_band_solve": (_i, [_i, View, View, _i64, _i64, _p, _p, _p, _p]),
    "lm_tri_solve": (_i, [_i, View, View, _i, _p, _p]),
    "lm_transpose_copy": (_i, [_i, View, View, _p]),
    "lm_diag_materialise": (_i, [_i, Vec, View, _p]),
    "lm_set_identity": (_i, [_i, View, _p]),
    "lm_lu_solve_batched": (_i, [_i, _i64, _i64, _p, _p, _p, _p, _p, _p]),
    "lm_solve_batched_classified": (_i, [_i, _i64, _i64, _p, _p, _p, _p, _p]),
    "lm_solve_batched_classified_from": (_i, [_i, _i64, _i64, _p, _p, _p, _p, _p, _p]),
    "lm_analyze_batched": (_i, [_i, _i64, _i64, _p, _p, _p]),
    "lm_expr_atb_schur_trace_batched": (_i, [_i, _i64, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "lm_fill_uniform": (_i, [_i, View, ctypes.c_uint64, _i64, _i64, _i64, _d, _d, _p]),
    "lm_fill_pcg64": (_i, [_i, _p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_uint64, ctypes.c_uint64,
                           ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _d, _d, _p]),
    "lm_nccl_load": (_i, [ctypes.c_char_p, ctypes.POINTER(_i)]),
    "lm_nccl_unique_id": (_i, [ctypes.c_char_p]),
    "lm_nccl_init_rank": (_i, [_i, _i, ctypes.c_char_p, ctypes.POINTER(_p)]),
    "lm_nccl_init_all": (_i, [_i, ctypes.POINTER(_i), ctypes.POINTER(_p)]),
    "lm_allreduce_sum": (_i, [_p, _i, _p, _i64, _p]),
    "lm_allreduce_sum_f64": (_i, [_p, _p, _p]),
    "lm_nccl_destroy": (_i, [_p]),
    "lm_debug_lu_panel": (_i, [View, _i64, _i, _p, _p, _p, _p]),
    "lm_debug_gemm_sub": (_i, [View, View, View, _p]),
}

_lock = threading.Lock()
_lib = None
_cuda_ok = None


def cuda_available() -> bool:
    """torch.cuda.is_available(), cached: it reads the environment on every
    call (~4 us), and every evaluate() asks several times."""
    global _cuda_ok
    if _cuda_ok is None:
        _cuda_ok = bool(torch.cuda.is_available())
    return _cuda_ok


def load_library(require_device: bool = True):
    """The ctypes handle; builds nothing.  ``require_device`` (default)
    refuses to run without a CUDA device."""
    global _lib
    if require_device and not cuda_available():
        raise BackendUnavailableError(
            "paper_2502_03000_b200 evaluates on a B200 (sm_100a) GPU only; no CUDA device is visible")
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise BackendUnavailableError(
                        f"C-ABI library not built ({LIB_PATH}); run `python -m paper_2502_03000_b200.build`")
                lib = ctypes.CDLL(str(LIB_PATH))
                for name, (res, args) in _SIGS.items():
                    f = getattr(lib, name)
                    f.restype = res
                    f.argtypes = args
                _lib = lib
    return _lib


def launch_count() -> int:
    return int(load_library(False).lm_launch_count()) if LIB_PATH.exists() else 0


def last_variant() -> str:
    """Kernel variant of this thread's last multi-variant call (lm_last_variant)."""
    return load_library(False).lm_last_variant().decode()


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise BackendError(f"unsupported element type {t.dtype}")


def _dev_check(t: torch.Tensor):
    if not t.is_cuda:
        raise BackendUnavailableError(
            "operand is not in device memory; this package has no CPU compute path")


def view(t: torch.Tensor) -> View:
    _dev_check(t)
    if t.dim() != 2:
        raise BackendError(f"2-D operand expected, got {t.dim()}-D")
    r, c = t.shape
    rs, cs = t.stride()
    return View(t.data_ptr(), r, c, rs, cs)


def vec(t: torch.Tensor) -> Vec:
    _dev_check(t)
    if t.dim() != 1:
        raise BackendError(f"1-D operand expected, got {t.dim()}-D")
    return Vec(t.data_ptr(), t.shape[0], t.stride(0))


def stream_handle(device=None) -> int:
    """Raw cudaStream_t of the current stream (torch's C binding: the Python
    torch.cuda.current_stream() wrapper costs ~10 us per call)."""
    if device is None:
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    return torch.cuda.current_stream(device).cuda_stream


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library(False).lm_last_error().decode(errors="replace")
        raise BackendError(f"{what} failed (rc={rc}): {msg}")


def call(name: str, *args) -> None:
    """Call a status-returning entry point on the current stream."""
    lib = load_library()
    rc = getattr(lib, name)(*args, ctypes.c_void_p(stream_handle()))
    check(rc, name)


def views(ts) -> ctypes.Array:
    arr = (View * max(len(ts), 1))()
    for k, t in enumerate(ts):
        arr[k] = view(t)
    return arr


def doubles(xs) -> ctypes.Array:
    xs = [float(x) for x in xs]
    return (ctypes.c_double * max(len(xs), 1))(*xs)
