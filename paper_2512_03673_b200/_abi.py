"""ctypes binding of the C-ABI declared in include/crt/convlinear4bit.h.

This is the same binding a maintainer of the reference would add (see
INTEGRATION.md); the torch-level mirror of the reference operator surface is
in ``api.py``.  There is no fallback: if libconvrot_b200.so cannot be loaded
the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libconvrot_b200.so")

# crt_status (errors.hpp:9-67 taxonomy)
CRT_OK = 0
CRT_ERR_INVALID_ORDER = 1
CRT_ERR_INVALID_VALUE = 2
CRT_ERR_SHAPE = 3
CRT_ERR_CAPACITY = 4
CRT_ERR_FORMAT = 5
CRT_ERR_CUDA = 6
CRT_ERR_UNSUPPORTED = 7
CRT_ERR_NCCL = 8
CRT_TP_COLUMN, CRT_TP_ROW = 1, 2

CRT_DTYPE_BF16, CRT_DTYPE_F32 = 0, 1
CRT_OUT_BF16, CRT_OUT_F32, CRT_OUT_I32_ACC = 0, 1, 2


class Error(RuntimeError):
    """Base class (convrot::Error, errors.hpp:9-13)."""
    status = -1


class InvalidOrderError(Error):
    status = CRT_ERR_INVALID_ORDER


class InvalidValueError(Error):
    status = CRT_ERR_INVALID_VALUE


class ShapeError(Error):
    status = CRT_ERR_SHAPE


class CapacityError(Error):
    status = CRT_ERR_CAPACITY


class FormatError(Error):
    status = CRT_ERR_FORMAT


class CudaError(Error):
    status = CRT_ERR_CUDA


class UnsupportedError(Error):
    status = CRT_ERR_UNSUPPORTED


class NcclError(Error):
    """NCCL unavailable or a collective failed (crt_tp_*; no reference
    counterpart: the reference is single-process)."""
    status = CRT_ERR_NCCL


_EXC = {c.status: c for c in (InvalidOrderError, InvalidValueError, ShapeError, CapacityError,
                              FormatError, CudaError, UnsupportedError, NcclError)}


class RotationSpecC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("group_size", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("identity_tail", ctypes.c_int32)]


class LayerDescC(ctypes.Structure):
    _fields_ = [("out_features", ctypes.c_int64), ("in_features", ctypes.c_int64),
                ("rotation", RotationSpecC), ("bits_w", ctypes.c_int32),
                ("w_dtype", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32

_SIGS = {
    "crt_abi_version": (_I32, []),
    "crt_last_error": (ctypes.c_char_p, []),
    "crt_launch_count": (_I64, []),
    "crt_debug_k1_trace": (None, [_P]),
    "crt_debug_k3_trace": (None, [_P]),
    "crt_regular_hadamard": (_I32, [_I32, _P]),
    "crt_sylvester_hadamard": (_I32, [_I32, _P]),
    "crt_rotate_quant": (_I32, [_P, _I32, _I64, _I64, _I64, ctypes.POINTER(RotationSpecC), _I32,
                                _P, _I64, _P, _P, _P]),
    "crt_rotated_row_absmax": (_I32, [_P, _I32, _I64, _I64, _I64, ctypes.POINTER(RotationSpecC),
                                      _P, _P]),
    "crt_layer_prepare": (_I32, [ctypes.POINTER(LayerDescC), _P, _I64, _P, _P,
                                 ctypes.POINTER(_P)]),
    "crt_layer_prepare_shard": (_I32, [ctypes.POINTER(LayerDescC), _P, _I64, _P, _I32, _I32, _P,
                                       ctypes.POINTER(_P)]),
    "crt_layer_from_codes": (_I32, [ctypes.POINTER(LayerDescC), _P, _I64, _P, _P, _P,
                                    ctypes.POINTER(_P)]),
    "crt_layer_destroy": (_I32, [_P]),
    "crt_layer_info": (_I32, [_P, ctypes.POINTER(LayerDescC)]),
    "crt_layer_export": (_I32, [_P, _P, _I64, _P, _P, _P]),
    "crt_rotate_quant_i8": (_I32, [_P, _I32, _I64, _I64, _I64, ctypes.POINTER(RotationSpecC), _P,
                                   _I64, _P, _P, _P]),
    "crt_quant_gemm_i8": (_I32, [_P, _I64, _P, _P, _P, _I64, _I32, _P, _I64, _P]),
    "crt_quant_gemm": (_I32, [_P, _I64, _P, _I32, _P, _I64, _I32, _P, _I64, _P]),
    "crt_layer_prepare_kshard": (_I32, [ctypes.POINTER(LayerDescC), _P, _I64, _P, _I32, _I32, _P,
                                        ctypes.POINTER(_P)]),
    "crt_rotate_quant_amax": (_I32, [_P, _I32, _I64, _I64, _I64, ctypes.POINTER(RotationSpecC),
                                     _P, _I32, _P, _I64, _P, _P, _P, _P]),
    "crt_dequant": (_I32, [_P, _I64, _I64, _P, _P, _I32, _P, _I64, _P]),
    "crt_workspace_create": (_I32, [_I64, _I64, ctypes.POINTER(_P)]),
    "crt_workspace_destroy": (_I32, [_P]),
    "crt_forward": (_I32, [_P, _P, _I32, _I64, _I64, _I32, _I32, _P, _I64, _P, _P]),
    "crt_forward_host": (_I32, [_P, _P, _I32, _I64, _I32, _I32, _P, _P, _P, _P, _P]),
    "crt_device_status": (_I32, [_P, _I32]),
    "crt_workspace_status": (_I32, [_P, _P, _I32]),
    "crt_nccl_unique_id": (_I32, [_P]),
    "crt_nccl_comm_create": (_I32, [_I32, _I32, _P, ctypes.POINTER(_P)]),
    "crt_nccl_comm_destroy": (_I32, [_P]),
    "crt_nccl_comm_info": (_I32, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "crt_tp_layer_prepare": (_I32, [ctypes.POINTER(LayerDescC), _P, _I64, _P, _I32, _P, _P,
                                    ctypes.POINTER(_P)]),
    "crt_tp_forward": (_I32, [_P, _P, _I32, _I64, _I64, _I32, _P, _I64, _I32, _P, _P, _P]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libconvrot_b200.so (building it in-tree first when the sources
    are newer and nvcc is available)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        from . import build as _build
        if build_if_missing and _build.needs_build():
            try:
                _build.build()
            except Exception as e:  # pragma: no cover - surfaced below
                if not os.path.exists(LIB_PATH):
                    raise ImportError(f"libconvrot_b200.so missing and build failed: {e}") from e
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libconvrot_b200.so not found at {LIB_PATH}; run "
                              "python -m paper_2512_03673_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.crt_abi_version() != 1:
            raise ImportError("ABI version mismatch")
        _lib = L
        return L


def check(status: int) -> None:
    if status != CRT_OK:
        msg = load().crt_last_error()
        msg = msg.decode() if msg else ""
        raise _EXC.get(status, Error)(msg)
