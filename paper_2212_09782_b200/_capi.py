"""ctypes binding of the C-ABI in include/qrtebd_c.h (libqrtebd_b200.so).

This is the FFI stub a Python host would write against the boundary; the
same declarations are what a cgo/JNI/N-API binding would carry
(INTEGRATION.md).  Loading fails loudly when the shared library is missing:
there is no CPU fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libqrtebd_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

QT_OK, QT_ERR_SHAPE, QT_ERR_INPUT, QT_ERR_NUMERIC, QT_ERR_CAPACITY, QT_ERR_CUDA, QT_ERR_NCCL, QT_ERR_INTERNAL = range(8)
SCHEME_SVD, SCHEME_EIG, SCHEME_QR, SCHEME_QR_CBE = range(4)
SCHEME_IDS = {"svd": 0, "eig": 1, "qr": 2, "qr_cbe": 3}


class qt_policy(C.Structure):
    _fields_ = [
        ("chi_max", C.c_uint64),
        ("sv_cutoff", C.c_double),
        ("target_eps", C.c_double),
        ("delta_chi_abs", C.c_uint64),
        ("delta_chi_rel", C.c_double),
        ("chi_max_expansion", C.c_uint64),
        ("qr_sweeps", C.c_int32),
        ("compute_explicit_error", C.c_int32),
        ("skip_renormalize", C.c_int32),
        ("reserved", C.c_int32),
    ]


class qt_report(C.Structure):
    _fields_ = [
        ("chi_before", C.c_uint64),
        ("chi_expanded", C.c_uint64),
        ("chi_after", C.c_uint64),
        ("eps_trunc", C.c_double),
        ("discarded_weight", C.c_double),
        ("scheme", C.c_int32),
        ("reserved", C.c_int32),
    ]


class qt_bond_report(C.Structure):
    _fields_ = [("bond", C.c_uint64), ("report", qt_report)]


class qt_isometry_report(C.Structure):
    _fields_ = [
        ("max_right_defect", C.c_double),
        ("max_left_defect", C.c_double),
        ("max_translation_defect", C.c_double),
        ("max_norm_defect", C.c_double),
        ("pass_", C.c_int32),
        ("reserved", C.c_int32),
    ]


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
U64P = C.POINTER(C.c_uint64)
DP = C.POINTER(C.c_double)

# name -> (restype, argtypes); every symbol declared in include/qrtebd_c.h
SIGNATURES = {
    "qt_last_error": (C.c_char_p, []),
    "qt_version": (C.c_char_p, []),
    "qt_policy_default": (None, [C.POINTER(qt_policy)]),
    "qt_expanded_dim": (C.c_uint64, [C.POINTER(qt_policy), C.c_uint64, C.c_uint64]),
    "qt_kernel_launches": (C.c_uint64, []),
    "qt_ctx_create": (C.c_int, [C.c_int, P, PP]),
    "qt_ctx_destroy": (C.c_int, [P]),
    "qt_ctx_synchronize": (C.c_int, [P]),
    "qt_ctx_stream": (P, [P]),
    "qt_ctx_set_qr_pair_min_rows": (C.c_int, [P, C.c_int64]),
    "qt_tensor_create": (C.c_int, [P, C.c_int, U64P, PP]),
    "qt_tensor_wrap": (C.c_int, [P, C.c_int, U64P, P, PP]),
    "qt_tensor_free": (C.c_int, [P]),
    "qt_tensor_shape": (C.c_int, [P, C.POINTER(C.c_int), U64P]),
    "qt_tensor_data": (P, [P]),
    "qt_tensor_upload": (C.c_int, [P, DP]),
    "qt_tensor_download": (C.c_int, [P, DP]),
    "qt_tensor_upload_async": (C.c_int, [P, DP]),
    "qt_tensor_download_async": (C.c_int, [P, DP]),
    "qt_tensor_copy": (C.c_int, [P, P]),
    "qt_qr_reduced": (C.c_int, [P, P, PP, PP]),
    "qt_lq_reduced": (C.c_int, [P, P, PP, PP]),
    "qt_zgemm": (C.c_int, [P, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                           P, C.c_int64, C.c_int64, P, C.c_int64, C.c_int64, P, C.c_int64, C.c_int64,
                           C.c_double, C.c_double]),
    "qt_apply_gate": (C.c_int, [P, C.c_int, P, P, P, P, C.POINTER(qt_policy), PP, PP, PP, PP,
                                C.POINTER(qt_report)]),
    "qt_apply_gate_qr": (C.c_int, [P, P, P, P, P, C.POINTER(qt_policy), PP, PP, PP, PP, C.POINTER(qt_report)]),
    "qt_apply_gate_qr_cbe": (C.c_int, [P, P, P, P, P, C.POINTER(qt_policy), PP, PP, PP, C.POINTER(qt_report)]),
    "qt_truncation_error_explicit": (C.c_int, [P, P, P, P, P, DP]),
    "qt_tebd_step_uniform": (C.c_int, [P, C.c_uint64, PP, PP, C.c_uint64, C.POINTER(C.c_int32), PP, C.c_int,
                                       C.POINTER(qt_policy), PP, PP, C.POINTER(qt_bond_report), U64P]),
    "qt_uniform_create": (C.c_int, [P, C.c_uint64, PP, PP, PP]),
    "qt_uniform_destroy": (C.c_int, [P]),
    "qt_uniform_step": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_int32), PP, C.c_int, C.POINTER(qt_policy), C.c_int32,
                                  C.POINTER(qt_bond_report), U64P]),
    "qt_uniform_view": (C.c_int, [P, C.c_int, C.c_uint64, PP]),
    "qt_finite_create": (C.c_int, [P, C.c_uint64, PP, C.c_uint64, P, PP]),
    "qt_finite_destroy": (C.c_int, [P]),
    "qt_finite_clone": (C.c_int, [P, PP]),
    "qt_finite_center_bond": (C.c_int, [P, U64P]),
    "qt_finite_view": (C.c_int, [P, C.c_int, C.c_uint64, PP]),
    "qt_finite_move_center": (C.c_int, [P, C.c_uint64]),
    "qt_finite_step": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_int32), PP, C.c_int, C.POINTER(qt_policy),
                                 C.POINTER(qt_bond_report), U64P]),
    "qt_finite_observables": (C.c_int, [P, P, DP, DP, C.c_uint64, U64P]),
    "qt_finite_step_observed": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_int32), PP, C.c_int, C.POINTER(qt_policy),
                                          C.POINTER(qt_bond_report), U64P, P, P]),
    "qt_nccl_get_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "qt_nccl_selftest": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_int)]),
    "qt_loopback_create": (C.c_int, [C.c_int, PP]),
    "qt_loopback_destroy": (C.c_int, [P]),
    "qt_chain_partition": (C.c_int, [C.c_uint64, C.c_int, C.c_int, U64P, U64P]),
    "qt_chain_create": (C.c_int, [P, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8), P, PP, PP, C.c_int, PP]),
    "qt_chain_destroy": (C.c_int, [P]),
    "qt_chain_range": (C.c_int, [P, U64P, U64P]),
    "qt_chain_view": (C.c_int, [P, C.c_int, C.c_uint64, PP]),
    "qt_tebd_step_finite_sharded": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_int32), PP, C.c_int,
                                              C.POINTER(qt_policy), C.POINTER(qt_bond_report), U64P]),
    "qt_left_defect": (C.c_int, [P, P, DP]),
    "qt_check_isometric_finite": (C.c_int, [P, C.c_double, DP, DP, DP, P]),
    "qt_expectation_local": (C.c_int, [P, P, P, P, DP]),
    "qt_schmidt_values": (C.c_int, [P, P, DP, U64P]),
    "qt_right_defect": (C.c_int, [P, P, DP]),
    "qt_check_isometric_uniform": (C.c_int, [P, C.c_uint64, PP, PP, C.c_double, DP, DP, DP, DP, P]),
    "qt_eigh": (C.c_int, [P, P, DP, PP]),
    "qt_bond_energy": (C.c_int, [P, P, P, P, P, DP]),
    "qt_fp64_peak": (C.c_int, [P, C.c_int, DP]),
    "qt_profile_begin": (C.c_int, [P, C.c_double]),
    "qt_profile_end": (C.c_int, [P, DP, DP, U64P]),
}

_lib = None


def load():
    """Load libqrtebd_b200.so; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("QRTEBD_B200_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise RuntimeError(
            f"{LIB_NAME} not found at {path}: build it with `make -C paper_2212_09782_b200` "
            "(there is no CPU fallback)")
    # the sharded chain resolves NCCL at run time: point it at torch's bundled
    # build (if any) so that a later `import torch` finds the same library
    if "QRTEBD_NCCL_LIB" not in os.environ:
        import sysconfig
        cand = Path(sysconfig.get_paths()["purelib"]) / "nvidia" / "nccl" / "lib" / "libnccl.so.2"
        if cand.exists():
            os.environ["QRTEBD_NCCL_LIB"] = str(cand)
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class QrtebdError(RuntimeError):
    """Base of the reference error taxonomy (proj/include/qrtebd/errors.hpp)."""

    status = QT_ERR_INTERNAL


class ShapeError(QrtebdError, ValueError):
    status = QT_ERR_SHAPE


class InputError(QrtebdError, ValueError):
    status = QT_ERR_INPUT


class NumericError(QrtebdError):
    status = QT_ERR_NUMERIC


class CapacityError(QrtebdError):
    status = QT_ERR_CAPACITY


class CudaError(QrtebdError):
    status = QT_ERR_CUDA


_ERRORS = {QT_ERR_SHAPE: ShapeError, QT_ERR_INPUT: InputError, QT_ERR_NUMERIC: NumericError,
           QT_ERR_CAPACITY: CapacityError, QT_ERR_CUDA: CudaError}


def check(status: int):
    if status != QT_OK:
        msg = load().qt_last_error().decode(errors="replace")
        raise _ERRORS.get(status, QrtebdError)(msg)


def default_policy(**kw) -> qt_policy:
    p = qt_policy()
    load().qt_policy_default(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise AttributeError(k)
        setattr(p, k, int(v) if isinstance(v, bool) else v)
    return p


class Context:
    """One CUDA device + stream + device workspace (qt_ctx)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load()
        h = C.c_void_p()
        check(self.lib.qt_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.qt_ctx_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def synchronize(self):
        check(self.lib.qt_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        return self.lib.qt_ctx_stream(self.h) or 0

    # ---- tensors
    def tensor(self, arr) -> "DeviceTensor":
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.complex128))
        return DeviceTensor.upload(self, a)

    def empty(self, shape) -> "DeviceTensor":
        shp = (C.c_uint64 * max(1, len(shape)))(*shape)
        h = C.c_void_p()
        check(self.lib.qt_tensor_create(self.h, len(shape), shp, C.byref(h)))
        return DeviceTensor(self, h)

    def wrap(self, ptr: int, shape) -> "DeviceTensor":
        shp = (C.c_uint64 * max(1, len(shape)))(*shape)
        h = C.c_void_p()
        check(self.lib.qt_tensor_wrap(self.h, len(shape), shp, C.c_void_p(ptr), C.byref(h)))
        return DeviceTensor(self, h)

    def fp64_peak(self, kind: int = 0) -> float:
        v = C.c_double()
        check(self.lib.qt_fp64_peak(self.h, kind, C.byref(v)))
        return v.value


class DeviceTensor:
    """Owned handle of a device-resident complex128 tensor (qt_tensor)."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.h = handle

    @classmethod
    def upload(cls, ctx: Context, a: np.ndarray) -> "DeviceTensor":
        t = ctx.empty(a.shape)
        check(ctx.lib.qt_tensor_upload(t.h, a.ctypes.data_as(DP)))
        return t

    @property
    def shape(self):
        r = C.c_int()
        s = (C.c_uint64 * 4)()
        check(self.ctx.lib.qt_tensor_shape(self.h, C.byref(r), s))
        return tuple(int(s[k]) for k in range(r.value))

    @property
    def ptr(self) -> int:
        return self.ctx.lib.qt_tensor_data(self.h) or 0

    def numpy(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=np.complex128)
        check(self.ctx.lib.qt_tensor_download(self.h, out.ctypes.data_as(DP)))
        return out

    def free(self):
        if self.h:
            check(self.ctx.lib.qt_tensor_free(self.h))
            self.h = None

    def __del__(self):
        try:
            if self.h and self.ctx.h:
                self.ctx.lib.qt_tensor_free(self.h)
        except Exception:
            pass
        self.h = None
