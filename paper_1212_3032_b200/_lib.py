"""ctypes binding of ``libewbem_b200.so`` (C ABI in ``include/ewbem_b200.h``).

The product path has no CPU fallback: importing a compute entry point
without the built library, or without a CUDA device, raises
:class:`NativeUnavailable` loudly.  Build with ``python -m
paper_1212_3032_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_NAME = "libewbem_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME

# Every symbol include/ewbem_b200.h declares (checked by tests/test_host.py).
EXPORTS = (
    "ewb_abi_version", "ewb_last_error", "ewb_launch_count", "ewb_ctx_create", "ewb_ctx_destroy",
    "ewb_ctx_set_exterior", "ewb_ctx_counts", "ewb_ctx_pair_lists", "ewb_static_rowsums", "ewb_static_tu",
    "ewb_assemble_tu",
    "ewb_assemble_system", "ewb_assemble_system_multi", "ewb_ctx_flags", "ewb_ctx_flags_async", "ewb_apply_bcs", "ewb_blockdiag_inverse",
    "ewb_gemv_batched", "ewb_set_solver_ctas", "ewb_solver_ctas",
    "ewb_gmres_workspace_bytes", "ewb_gmres",
    "ewb_sem_workspace_bytes", "ewb_sem_guess", "ewb_sem_from_products",
    "ewb_opgmres_workspace_bytes", "ewb_opgmres_buffers", "ewb_opgmres_phase", "ewb_window_idft",
    "ewb_matfree_workspace_bytes", "ewb_matfree_apply", "ewb_matfree_apply_masked",
    "ewb_pair_kernels_blocks", "ewb_pair_kernels_workspace_bytes",
    "ewb_pair_kernels_reduce", "ewb_fp64_peak_probe", "ewb_debug_checks",
    "ewb_math_selftest", "ewb_math_selftest_delta",
)

EWB_OK, EWB_ERR_INVALID, EWB_ERR_CUDA, EWB_ERR_NONFINITE = 0, 1, 2, 3
ABI_VERSION = 6


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing: there is no fallback."""


class NativeError(RuntimeError):
    pass


class GmresResult(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("n_hist", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("matvecs", ctypes.c_int32),
                ("init_residual", ctypes.c_double), ("final_residual", ctypes.c_double)]


_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
D = ctypes.c_double

_SIGS = {
    "ewb_abi_version": (I32, []),
    "ewb_last_error": (ctypes.c_char_p, []),
    "ewb_launch_count": (I64, []),
    "ewb_ctx_create": (I32, [P, P, P, P, P, I64, D, D, D, P, P, P, P, P, P, ctypes.POINTER(P)]),
    "ewb_ctx_destroy": (I32, [P]),
    "ewb_ctx_counts": (I32, [P, P]),
    "ewb_ctx_set_exterior": (I32, [P, I32, P]),
    "ewb_ctx_pair_lists": (I32, [P, P, P, P, P, P, P]),
    "ewb_static_rowsums": (I32, [P, P, P]),
    "ewb_static_tu": (I32, [P, P, P, P]),
    "ewb_assemble_tu": (I32, [P, D, D, P, P, P]),
    "ewb_assemble_system": (I32, [P, D, D, P, P, P, P, P, P]),
    "ewb_assemble_system_multi": (I32, [P, I32, P, P, P, P, P, P, P, P, P]),
    "ewb_ctx_flags": (I32, [P, P, P, P]),
    "ewb_ctx_flags_async": (I32, [P, P, P]),
    "ewb_apply_bcs": (I32, [P, P, P, P, I64, P, P, P]),
    "ewb_blockdiag_inverse": (I32, [P, I64, P, P, P]),
    "ewb_gemv_batched": (I32, [P, P, P, I64, I32, P]),
    "ewb_set_solver_ctas": (I32, [I32]),
    "ewb_solver_ctas": (I32, []),
    "ewb_gmres_workspace_bytes": (I64, [I64, I32]),
    "ewb_gmres": (I32, [P, P, P, P, I32, P, I64, D, I32, I32, P, I64, P, I32, P, P]),
    "ewb_sem_workspace_bytes": (I64, [I64, I32]),
    "ewb_sem_guess": (I32, [P, P, P, I32, I64, D, P, P, P, I64, P, P]),
    "ewb_sem_from_products": (I32, [P, P, P, I32, I64, D, P, P, P, I64, P, P]),
    "ewb_opgmres_workspace_bytes": (I64, [I64, I32]),
    "ewb_opgmres_buffers": (I32, [P, I64, I32, P, P, P, P, P, P]),
    "ewb_opgmres_phase": (I32, [I32, P, I64, P, P, I32, P, P, P, I32, I64, D, I32, I32, P, I32,
                                P]),
    "ewb_window_idft": (I32, [P, I64, I64, I32, D, D, P, P, P]),
    "ewb_matfree_workspace_bytes": (I64, [P, I32]),
    "ewb_matfree_apply": (I32, [P, D, D, P, P, I32, P, P, P, P, I64, P, P]),
    "ewb_matfree_apply_masked": (I32, [P, D, D, P, P, I32, ctypes.c_uint32, ctypes.c_uint32, P, P,
                                       P, P, I64, P, P]),
    "ewb_pair_kernels_blocks": (I32, [P, I64, P, I64, P, I32, D, D, D, P, P, P]),
    "ewb_pair_kernels_workspace_bytes": (I64, [I64, I64, I32]),
    "ewb_pair_kernels_reduce": (I32, [P, I64, P, I64, P, P, I32, D, D, D, P, P, P, I64, P]),
    "ewb_fp64_peak_probe": (I32, [I64, I32, P, P, P]),
    "ewb_debug_checks": (I32, [P, P, I32]),
    "ewb_math_selftest": (I32, [P, I64, P, P, P, P]),
    "ewb_math_selftest_delta": (I32, [P, I64, P, P]),
}


def load(path: os.PathLike | None = None):
    """Load (once) and return the ctypes library.  Raises NativeUnavailable.

    ``EWB_LIBRARY`` selects another build of the same ABI (the debug-check
    build of DESIGN.md §4, ``paper_1212_3032_b200/variants/debug.so``)."""
    global _lib
    if _lib is not None:
        return _lib
    env = os.environ.get("EWB_LIBRARY")
    p = Path(path) if path else (Path(env) if env else LIB_PATH)
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is not built; run `python -m paper_1212_3032_b200.build` "
            "(there is no CPU fallback for the B200 path)")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None and p != LIB_PATH:
            continue   # an older A/B build (tools/build_variant.py) without this entry point
        if fn is None:
            raise NativeUnavailable(f"{p} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    if lib.ewb_abi_version() != ABI_VERSION:
        raise NativeUnavailable("libewbem_b200.so ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == EWB_OK:
        return
    msg = load().ewb_last_error().decode(errors="replace")
    if rc == EWB_ERR_INVALID:
        raise ValueError(msg)
    if rc == EWB_ERR_NONFINITE:
        raise FloatingPointError(msg)
    raise NativeError(f"{what}: {msg}" if what else msg)


def require_cuda():
    """The library plus a CUDA device, or NativeUnavailable."""
    import torch

    lib = load()
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return lib


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (must be contiguous)."""
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
