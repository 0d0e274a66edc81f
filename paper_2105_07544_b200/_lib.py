"""ctypes binding of libmpkb200.so (the C ABI in include/mpk_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_2105_07544_b200.build``.  There is no CPU fallback: if the
library is missing, or no CUDA device is present, every device operation
raises :class:`NativeUnavailable` loudly.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MPK_LIB_PATH: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("MPK_LIB_PATH") or os.path.join(HERE, "_lib", "libmpkb200.so")

F32, F64 = 0, 1
CSR, STENCIL = 0, 1
PRESET_IDS = {"Laplace2D": 0, "Laplace3D": 1, "UniFlow2D": 2, "BentPipe2D": 3, "Stretched2D": 4}
PC_NONE, PC_JACOBI, PC_POLY = 0, 1, 2
RULE_NU, RULE_U = 0, 1
MAX_STEPS = 512

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = (
    "mpk_abi_version", "mpk_last_error", "mpk_sm_count", "mpk_spmv", "mpk_convert",
    "mpk_reduce_ws_bytes", "mpk_dot", "mpk_norm2", "mpk_axpy", "mpk_scale", "mpk_cgs2_append",
    "mpk_cycle_hess_bytes", "mpk_cycle_run", "mpk_residual", "mpk_ir_update",
    "mpk_precond_apply", "mpk_prof_reset", "mpk_prof_read", "mpk_lsq_init", "mpk_lsq_update",
    "mpk_lsq_solve", "mpk_vdiv", "mpk_launch_count", "mpk_fused_prof_read", "mpk_comm_part_bytes",
    "mpk_dev_alloc", "mpk_dev_free", "mpk_ipc_get", "mpk_ipc_open", "mpk_ipc_close", "mpk_rcm_host",
    "mpk_last_cycle_kernel", "mpk_can_access_peer", "mpk_comm_push_rows", "mpk_comm_reduce_ctl",
    "mpk_block_lu", "mpk_stencil_assemble", "mpk_stencil_assemble_ws_bytes", "mpk_l2_release",
)
MAX_RANKS = 8


class NativeUnavailable(RuntimeError):
    """The sm_100a library (or a CUDA device) is not available."""


ABI_VERSION = 2   # include/mpk_b200.h MPK_ABI_VERSION


class MpkMatrix(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("dtype", ctypes.c_int32), ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
        ("values", ctypes.c_void_p), ("preset", ctypes.c_int32), ("nx", ctypes.c_int32),
        ("row0", ctypes.c_int64), ("diffusion", ctypes.c_double), ("velocity", ctypes.c_double),
        ("convection", ctypes.c_double), ("stretch", ctypes.c_double), ("band", ctypes.c_int64),
    ]


class MpkPrecond(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("dtype", ctypes.c_int32), ("n", ctypes.c_int64),
        ("block", ctypes.c_int32), ("lu", ctypes.c_void_p), ("piv", ctypes.c_void_p),
        ("degree", ctypes.c_int32), ("roots_re", ctypes.POINTER(ctypes.c_double)),
        ("roots_im", ctypes.POINTER(ctypes.c_double)), ("poly_A", ctypes.POINTER(MpkMatrix)),
        ("work", ctypes.c_void_p),
    ]


class MpkCycleCtl(ctypes.Structure):
    _fields_ = [
        ("done", ctypes.c_int32), ("steps", ctypes.c_int32), ("breakdown", ctypes.c_int32),
        ("tri_err", ctypes.c_int32), ("tri_index", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("tri_entry", ctypes.c_double), ("tri_threshold", ctypes.c_double),
        ("gamma", ctypes.c_double), ("scale", ctypes.c_double),
        ("implicit_relres", ctypes.c_double * MAX_STEPS),
    ]


class MpkComm(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("ctas", ctypes.c_int32),
        ("pad_", ctypes.c_int32), ("row0", ctypes.c_int64),
        ("part", ctypes.c_void_p * MAX_RANKS), ("xbar", ctypes.c_void_p * MAX_RANKS),
        ("epoch", ctypes.c_void_p), ("xg", ctypes.c_void_p * MAX_RANKS),
        ("mir_lo", ctypes.c_int64 * MAX_RANKS), ("mir_hi", ctypes.c_int64 * MAX_RANKS),
    ]


class MpkCycleDesc(ctypes.Structure):
    _fields_ = [
        ("A", ctypes.POINTER(MpkMatrix)), ("M", ctypes.POINTER(MpkPrecond)),
        ("dtype", ctypes.c_int32), ("m", ctypes.c_int32), ("steps_cap", ctypes.c_int32),
        ("rule", ctypes.c_int32), ("exit_tol", ctypes.c_double), ("norm_scale", ctypes.c_double),
        ("n", ctypes.c_int64), ("ld", ctypes.c_int64), ("V", ctypes.c_void_p),
        ("r0", ctypes.c_void_p), ("rnorm2", ctypes.c_void_p), ("x0", ctypes.c_void_p),
        ("x_out", ctypes.c_void_p), ("work", ctypes.c_void_p), ("hess", ctypes.c_void_p),
        ("ws", ctypes.c_void_p), ("ctl", ctypes.c_void_p), ("nranks", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("comm", ctypes.POINTER(MpkComm)),
    ]


_LIB = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32

_SIGS = {
    "mpk_abi_version": (_I32, []),
    "mpk_last_error": (ctypes.c_char_p, []),
    "mpk_sm_count": (_I32, []),
    "mpk_spmv": (_I32, [ctypes.POINTER(MpkMatrix), _P, _P, _P]),
    "mpk_convert": (_I32, [_I32, _I32, _I64, _P, _P, _P]),
    "mpk_reduce_ws_bytes": (_I64, [_I64, _I32]),
    "mpk_dot": (_I32, [_I32, _I64, _P, _P, _P, _P, _P]),
    "mpk_norm2": (_I32, [_I32, _I64, _P, _P, _P, _P]),
    "mpk_axpy": (_I32, [_I32, _I64, ctypes.c_double, _P, _P, _P, _P]),
    "mpk_scale": (_I32, [_I32, _I64, ctypes.c_double, _P, _P, _P]),
    "mpk_cgs2_append": (_I32, [_I32, _I64, _I64, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P]),
    "mpk_cycle_hess_bytes": (_I64, [_I32, _I32]),
    "mpk_cycle_run": (_I32, [ctypes.POINTER(MpkCycleDesc), _P]),
    "mpk_residual": (_I32, [ctypes.POINTER(MpkMatrix), _P, _P, _P, _P, _P, _P, _P, _P]),
    "mpk_ir_update": (_I32, [_I64, _P, _P, _P, _P]),
    "mpk_precond_apply": (_I32, [ctypes.POINTER(MpkPrecond), _P, _P, _P]),
    "mpk_prof_reset": (_I32, []),
    "mpk_prof_read": (_I32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                             ctypes.POINTER(ctypes.c_double), _I32]),
}
_SIGS["mpk_launch_count"] = (_I64, [])
_SIGS["mpk_last_cycle_kernel"] = (ctypes.c_char_p, [])
_SIGS["mpk_can_access_peer"] = (_I32, [_I32, _I32])
_SIGS["mpk_l2_release"] = (_I32, [])
_SIGS["mpk_comm_push_rows"] = (_I32, [ctypes.c_void_p, _I32, _I64, _P, _P])
_SIGS["mpk_comm_reduce_ctl"] = (_I32, [ctypes.c_void_p, _I32, _P, _I32, _I32, _P])
_SIGS["mpk_fused_prof_read"] = (_I32, [ctypes.POINTER(ctypes.c_uint64), _I32])
_SIGS["mpk_comm_part_bytes"] = (_I64, [_I32])
_SIGS["mpk_dev_alloc"] = (_I32, [_I64, ctypes.POINTER(ctypes.c_void_p)])
_SIGS["mpk_dev_free"] = (_I32, [_P])
_SIGS["mpk_ipc_get"] = (_I32, [_P, _P])
_SIGS["mpk_ipc_open"] = (_I32, [_P, ctypes.POINTER(ctypes.c_void_p)])
_SIGS["mpk_ipc_close"] = (_I32, [_P])
_SIGS["mpk_rcm_host"] = (_I32, [_I64, _P, _P, _P])
_SIGS["mpk_vdiv"] = (_I32, [_I32, _I64, _P, _P, _P, _P])
_SIGS["mpk_lsq_init"] = (_I32, [_I32, _I32, ctypes.c_double, ctypes.c_double, _P, _P, _P])
_SIGS["mpk_lsq_update"] = (_I32, [_I32, _I32, _I32, _P, _P, _P, _P, _P, _P])
_SIGS["mpk_lsq_solve"] = (_I32, [_I32, _I32, _I32, _P, _P, _P])
_SIGS["mpk_block_lu"] = (_I32, [ctypes.POINTER(MpkMatrix), _I32, _P, _P, _P, _P, _P, _P])
_SIGS["mpk_stencil_assemble"] = (_I32, [ctypes.POINTER(MpkMatrix), _P, _P, _P, _P, _P])
_SIGS["mpk_stencil_assemble_ws_bytes"] = (_I64, [_I64])


def load(require_device: bool = True):
    """Load the library (once).  Raises NativeUnavailable when it cannot run."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                "libmpkb200.so not built (%s); run __graft_entry__.build()" % LIB_PATH)
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.mpk_abi_version() != ABI_VERSION:
            raise NativeUnavailable("libmpkb200.so has ABI %d, this package needs %d: rebuild it"
                                    % (lib.mpk_abi_version(), ABI_VERSION))
        _LIB = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return _LIB


def last_cycle_kernel() -> str:
    """Kernel family of this thread's last mpk_cycle_run (tests prove dispatch with it)."""
    return load(require_device=False).mpk_last_cycle_kernel().decode()


def check(rc: int):
    if rc != 0:
        msg = _LIB.mpk_last_error().decode(errors="replace") if _LIB is not None else ""
        raise RuntimeError("libmpkb200 error %d: %s" % (rc, msg))
