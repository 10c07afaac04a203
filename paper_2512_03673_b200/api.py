"""Torch-level mirror of the reference operator surface for the
ConvLinear4bit path (reference: /root/reference/proj/core/include/convrot/
{hadamard,quant,pipeline}.hpp).  Names, argument meaning and error classes
follow the reference; tensors are CUDA tensors and every call goes through
the C-ABI (``_abi.py`` -> libconvrot_b200.so).  PyTorch only supplies device
memory and the current stream.
"""
from __future__ import annotations

import ctypes
import threading
import enum
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _abi
from ._abi import (CapacityError, CudaError, Error, FormatError, InvalidOrderError,  # noqa: F401
                   InvalidValueError, ShapeError, UnsupportedError, check)


class RotationKind(enum.IntEnum):
    """pipeline.hpp:14 (random_orthogonal is out of scope here)."""
    none = 0
    sylvester = 1
    regular = 2


@dataclass(frozen=True)
class RotationSpec:
    """pipeline.hpp:23-30.  group_size 0 = global (one block over K)."""
    kind: RotationKind = RotationKind.none
    group_size: int = 0
    seed: int = 0
    identity_tail: bool = False

    def c(self) -> _abi.RotationSpecC:
        return _abi.RotationSpecC(int(self.kind), int(self.group_size), int(self.seed),
                                  int(self.identity_tail))


@dataclass(frozen=True)
class QuantSpec:
    """quant.hpp:15-20: symmetric per-row quantizer, codes in [-qmax, qmax]."""
    bits: int = 4

    def qmax(self) -> int:
        return (1 << (self.bits - 1)) - 1


_OUT = {"bf16": _abi.CRT_OUT_BF16, "f32": _abi.CRT_OUT_F32, "i32": _abi.CRT_OUT_I32_ACC}
_OUT_DTYPE = {"bf16": torch.bfloat16, "f32": torch.float32, "i32": torch.int32}


def _lib():
    return _abi.load()


def _stream(t: Optional[torch.Tensor] = None) -> ctypes.c_void_p:
    dev = t.device if t is not None else torch.device("cuda")
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _abi.CRT_DTYPE_BF16
    if t.dtype == torch.float32:
        return _abi.CRT_DTYPE_F32
    raise InvalidValueError(f"unsupported input dtype {t.dtype} (bf16 or f32)")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check_2d_cuda(x: torch.Tensor, what: str) -> None:
    if not x.is_cuda:
        raise InvalidValueError(f"{what} must be a CUDA tensor")
    if x.dim() != 2:
        raise ShapeError(f"{what} must be 2-D")
    if x.stride(1) != 1:
        raise ShapeError(f"{what} must be row-major with unit column stride")


# ---------------------------------------------------------------------------
# a1: Hadamard construction (hadamard.cpp:70-126)
# ---------------------------------------------------------------------------
def regular(n: int) -> np.ndarray:
    """Regular Hadamard sign matrix H_n = H4^{(x)log4 n} (hadamard.cpp:91-106)."""
    out = np.empty((n, n) if 0 < n <= 4096 else (1,), np.int8)
    check(_lib().crt_regular_hadamard(n, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def sylvester(n: int) -> np.ndarray:
    out = np.empty((n, n) if 0 < n <= 4096 else (1,), np.int8)
    check(_lib().crt_sylvester_hadamard(n, out.ctypes.data_as(ctypes.c_void_p)))
    return out


# ---------------------------------------------------------------------------
# K1: group_rotate -> compute_scales -> quantize -> pack_int4
# ---------------------------------------------------------------------------
def packed_row_bytes(k: int, bits: int) -> int:
    return (k + 1) // 2 if bits == 4 else k


def rotate_quantize(x: torch.Tensor, rotation: RotationSpec, aq: QuantSpec = QuantSpec(4),
                    *, scales64: bool = False, check_finite: bool = True):
    """Fused group_rotate + compute_scales + quantize + pack_int4 on the GPU.

    Returns ``(codes, scales_f32[, scales_f64])``: codes is uint8
    [M, ld] with the reference nibble layout in the first ceil(K/2) bytes of
    each row (bits 4) or int8 codes (bits 8).  Bit-identical to the
    reference's quantize(group_rotate(x)) codes and compute_scales."""
    _check_2d_cuda(x, "x")
    M, K = x.shape
    row = packed_row_bytes(K, aq.bits)
    ld = max(16, (row + 15) // 16 * 16)
    codes = torch.empty((M, ld), dtype=torch.uint8, device=x.device)
    s32 = torch.empty(M, dtype=torch.float32, device=x.device)
    s64 = torch.empty(M, dtype=torch.float64, device=x.device) if scales64 else None
    rc = rotation.c()
    st = _stream(x)
    check(_lib().crt_rotate_quant(_ptr(x), _dtype_code(x), M, K, x.stride(0), ctypes.byref(rc),
                                  aq.bits, _ptr(codes), ld, _ptr(s32), _ptr(s64), st))
    if check_finite:
        check(_lib().crt_device_status(st, 1))
    return (codes, s32, s64) if scales64 else (codes, s32)


def rotate_quantize_into(x: torch.Tensor, rotation: RotationSpec, codes: torch.Tensor,
                         scales: torch.Tensor, aq: QuantSpec = QuantSpec(4),
                         scales64: Optional[torch.Tensor] = None) -> None:
    """rotate_quantize into caller-owned buffers (no allocation, no sync):
    codes uint8 [M, ld] with ld >= packed row bytes, scales fp32 [M]."""
    _check_2d_cuda(x, "x")
    M, K = x.shape
    if codes.shape[0] < M or codes.stride(1) != 1 or scales.numel() < M:
        raise ShapeError("rotate_quantize_into: output buffers too small")
    rc = rotation.c()
    check(_lib().crt_rotate_quant(_ptr(x), _dtype_code(x), M, K, x.stride(0), ctypes.byref(rc),
                                  aq.bits, _ptr(codes), codes.stride(0), _ptr(scales),
                                  _ptr(scales64), _stream(x)))


# ---------------------------------------------------------------------------
# K2: prepare_layer (pipeline.cpp:158-176)
# ---------------------------------------------------------------------------
class PreparedLayer:
    """Offline-rotated, offline-quantized weights (pipeline.hpp:55-65), owned
    on the device by an immutable C-ABI handle."""

    def __init__(self, handle: int, out_features: int, in_features: int, rotation: RotationSpec,
                 weight_quant: QuantSpec, has_bias: bool, name: str, device: torch.device,
                 shard: Tuple[int, int] = (0, 1)):
        self._h = ctypes.c_void_p(handle)
        self.out_features = out_features
        self.in_features = in_features
        self.rotation = rotation
        self.weight_quant = weight_quant
        self.has_bias = has_bias
        self.name = name
        self.device = device
        self.shard = shard

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None or not self._h.value:
            raise Error("layer destroyed")
        return self._h

    def export(self, scales64: bool = True):
        """(codes [N, ceil(K/2)] uint8 packed like pack_int4 (or int8 rows for
        8-bit), scales f32, scales f64) -- the reference layout."""
        N, K = self.out_features, self.in_features
        row = packed_row_bytes(K, self.weight_quant.bits)
        codes = torch.empty((N, max(row, 1)), dtype=torch.uint8, device=self.device)
        s32 = torch.empty(N, dtype=torch.float32, device=self.device)
        s64 = torch.empty(N, dtype=torch.float64, device=self.device) if scales64 else None
        with torch.cuda.device(self.device):
            check(_lib().crt_layer_export(self.handle, _ptr(codes), max(row, 1), _ptr(s32),
                                          _ptr(s64), _stream()))
        return (codes[:, :row], s32, s64) if scales64 else (codes[:, :row], s32)

    def close(self) -> None:
        if self._h is not None and self._h.value:
            _lib().crt_layer_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _prepare(w, bias, rotation, wq, name, rank, nranks, kshard=False):
    _check_2d_cuda(w, "w")
    if not w.is_contiguous() and w.stride(1) != 1:
        raise ShapeError("w must be row-major")
    N, K = w.shape
    if bias is not None:
        if bias.numel() != N:  # pipeline.cpp:162-164
            raise ShapeError("prepare_layer: bias length must equal out_features")
        bias = bias.to(device=w.device, dtype=torch.float32).contiguous()
    desc = _abi.LayerDescC(N, K, rotation.c(), wq.bits, _dtype_code(w))
    h = ctypes.c_void_p()
    with torch.cuda.device(w.device):
        st = _stream(w)
        if kshard:
            check(_lib().crt_layer_prepare_kshard(ctypes.byref(desc), _ptr(w), w.stride(0),
                                                  _ptr(bias), rank, nranks, st, ctypes.byref(h)))
        elif nranks == 1:
            check(_lib().crt_layer_prepare(ctypes.byref(desc), _ptr(w), w.stride(0), _ptr(bias),
                                           st, ctypes.byref(h)))
        else:
            check(_lib().crt_layer_prepare_shard(ctypes.byref(desc), _ptr(w), w.stride(0),
                                                 _ptr(bias), rank, nranks, st, ctypes.byref(h)))
        # non-finite weights: the C-ABI reports them synchronously
        # (compute_scales throws, quant.cpp:16-18)
    if kshard:
        return PreparedLayer(h.value, N, K // nranks, rotation, wq, bias is not None, name,
                             w.device, (rank, nranks))
    return PreparedLayer(h.value, N // nranks, K, rotation, wq, bias is not None, name, w.device,
                         (rank, nranks))


def prepare_layer(w: torch.Tensor, bias: Optional[torch.Tensor], rotation: RotationSpec,
                  wq: QuantSpec = QuantSpec(4), name: str = "") -> PreparedLayer:
    return _prepare(w, bias, rotation, wq, name, 0, 1)


def prepare_layer_shard(w: torch.Tensor, bias: Optional[torch.Tensor], rotation: RotationSpec,
                        wq: QuantSpec, rank: int, nranks: int, name: str = "") -> PreparedLayer:
    """Column-parallel shard: output channels [rank*N/P, (rank+1)*N/P)."""
    return _prepare(w, bias, rotation, wq, name, rank, nranks)


def prepare_layer_kshard(w: torch.Tensor, bias: Optional[torch.Tensor], rotation: RotationSpec,
                         wq: QuantSpec, rank: int, nranks: int, name: str = "") -> PreparedLayer:
    """Row-parallel shard: input columns [rank*K/P, (rank+1)*K/P) of the full
    layer's codes, with the full layer's per-channel scales and bias."""
    return _prepare(w, bias, rotation, wq, name, rank, nranks, kshard=True)


# ---------------------------------------------------------------------------
# K3 + forward (pipeline.cpp:178-233)
# ---------------------------------------------------------------------------
class Workspace:
    """Activation codes/scales scratch for forward (no hidden allocations)."""

    def __init__(self, max_m: int, max_k: int, device=None):
        self.max_m, self.max_k = max_m, max_k
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(_lib().crt_workspace_create(max_m, max_k, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def status(self, reset: bool = True) -> None:
        """Raise InvalidValueError if a forward run with this workspace saw a
        non-finite input (its own error word; synchronises the stream)."""
        with torch.cuda.device(self.device):
            check(_lib().crt_workspace_status(self._h, _stream(), int(reset)))

    def close(self):
        if self._h is not None and self._h.value:
            _lib().crt_workspace_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


_ws_cache = {}
_ws_lock = threading.Lock()


def _workspace_for(M: int, K: int, device) -> Workspace:
    """The default workspace of (device, current stream): forwards on
    different streams never share activation-code scratch."""
    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    with _ws_lock:
        return _workspace_locked(key, M, K, device)


def _workspace_locked(key, M: int, K: int, device) -> Workspace:
    ws = _ws_cache.get(key)
    if ws is None or ws.max_m < M or ws.max_k < K:
        ws = Workspace(max(M, ws.max_m if ws else 0), max(K, ws.max_k if ws else 0), device)
        _ws_cache[key] = ws
    return ws


def _same_device(a, b) -> bool:
    a, b = torch.device(a), torch.device(b)
    if a.type != b.type:
        return False
    cur = torch.cuda.current_device() if a.type == "cuda" else 0
    return (cur if a.index is None else a.index) == (cur if b.index is None else b.index)


def _check_out(y: torch.Tensor, M: int, N: int, out: str, device) -> None:
    """A caller-supplied output buffer must be exactly what the kernels write:
    the out kind's dtype, [M, N] (row pitch >= N), unit column stride, on the
    layer's device."""
    if y.dtype != _OUT_DTYPE[out]:
        raise InvalidValueError(f"y must be {_OUT_DTYPE[out]} for out={out!r}, got {y.dtype}")
    if y.dim() != 2 or tuple(y.shape) != (M, N) or y.stride(1) != 1 or y.stride(0) < N:
        raise ShapeError(f"y must be a row-major [{M}, {N}] matrix, got {tuple(y.shape)} "
                         f"strides {y.stride()}")
    if not _same_device(y.device, device):
        raise InvalidValueError(f"y is on {y.device}, the layer on {device}")


def forward(x: torch.Tensor, layer: PreparedLayer, aq: QuantSpec = QuantSpec(4), *,
            out: str = "bf16", y: Optional[torch.Tensor] = None,
            workspace: Optional[Workspace] = None, check_finite: bool = True) -> torch.Tensor:
    """Online half of ConvLinear4bit (pipeline.cpp:206-233): rotate x,
    per-token quantize, integer GEMM against the prepared weights, dequantize
    by s_a[m]*s_w[n], add bias.  ``out``: "bf16" (production), "f32"
    (dequant parity) or "i32" (raw int_gemm accumulators).

    Non-finite input raises InvalidValueError like the reference
    (compute_scales, quant.cpp:16-18): with ``check_finite`` (default) the
    call synchronises the stream and reads the workspace's own error word.
    Pipelined callers pass ``check_finite=False`` and poll
    ``workspace.status()`` when convenient."""
    _check_2d_cuda(x, "x")
    M, K = x.shape
    if K != layer.in_features:  # pipeline.cpp:208-212
        raise ShapeError(f"forward: input has {K} columns, layer expects {layer.in_features}")
    if aq.bits not in (4, 8):  # :213-215
        raise InvalidValueError("forward: activation bits must be 4 or 8")
    if not _same_device(x.device, layer.device):
        raise InvalidValueError(f"x is on {x.device}, the layer on {layer.device}")
    N = layer.out_features
    if y is None:
        y = torch.empty((M, N), dtype=_OUT_DTYPE[out], device=x.device)
    else:
        _check_out(y, M, N, out, layer.device)
    ws = workspace or _workspace_for(M, K, x.device)
    if ws.max_m < M or ws.max_k < K:
        raise ShapeError("workspace too small")
    st = _stream(x)
    check(_lib().crt_forward(layer.handle, _ptr(x), _dtype_code(x), M, x.stride(0), aq.bits,
                             _OUT[out], _ptr(y), y.stride(0), ws.handle, st))
    if check_finite:
        check(_lib().crt_workspace_status(ws.handle, st, 1))
    return y


def quant_gemm(codes: torch.Tensor, scales: torch.Tensor, layer: PreparedLayer,
               aq: QuantSpec = QuantSpec(4), *, out: str = "bf16",
               y: Optional[torch.Tensor] = None) -> torch.Tensor:
    """int_gemm + dequant on pre-quantized activations (K1 output)."""
    M = codes.shape[0]
    N = layer.out_features
    if y is None:
        y = torch.empty((M, N), dtype=_OUT_DTYPE[out], device=codes.device)
    else:
        _check_out(y, M, N, out, layer.device)
    check(_lib().crt_quant_gemm(_ptr(codes), codes.stride(0), _ptr(scales), aq.bits, layer.handle,
                                M, _OUT[out], _ptr(y), y.stride(0), _stream(codes)))
    return y


def rotate_quantize_i8(x: torch.Tensor, rotation: RotationSpec):
    """K1 for the hardware-expansion GEMM: 4-bit codes stored one int8 per
    code ([M, ld] uint8 holding -7..7 as int8), fp32 scales and the per-row
    code sums (int32)."""
    _check_2d_cuda(x, "x")
    M, K = x.shape
    ld = max(16, (K + 15) // 16 * 16)
    codes = torch.empty((M, ld), dtype=torch.uint8, device=x.device)
    s32 = torch.empty(M, dtype=torch.float32, device=x.device)
    sums = torch.empty(M, dtype=torch.int32, device=x.device)
    rc = rotation.c()
    check(_lib().crt_rotate_quant_i8(_ptr(x), _dtype_code(x), M, K, x.stride(0), ctypes.byref(rc),
                                     _ptr(codes), ld, _ptr(s32), _ptr(sums), _stream(x)))
    return codes, s32, sums


def rotate_quantize_amax(x: torch.Tensor, rotation: RotationSpec, amax: torch.Tensor,
                         int8_codes: bool = True, bits: int = 4):
    """K1 on a column shard with the GLOBAL exact per-row maxima ``amax``
    (float64, device): returns (codes, fp32 scales, code sums or None).
    int8_codes: the crt_quant_gemm_i8 layout (bits 4 only); else packed."""
    _check_2d_cuda(x, "x")
    M, K = x.shape
    if amax.dtype != torch.float64 or amax.numel() != M or not amax.is_contiguous():
        raise ShapeError("amax must be a contiguous float64 vector of M rows")
    if int8_codes and bits != 4:
        raise InvalidValueError("int8-stored codes are for 4-bit activations")
    row = K if (int8_codes or bits == 8) else (K + 1) // 2
    ld = max(16, (row + 15) // 16 * 16)
    codes = torch.empty((M, ld), dtype=torch.uint8, device=x.device)
    s32 = torch.empty(M, dtype=torch.float32, device=x.device)
    sums = torch.empty(M, dtype=torch.int32, device=x.device) if int8_codes else None
    rc = rotation.c()
    check(_lib().crt_rotate_quant_amax(_ptr(x), _dtype_code(x), M, K, x.stride(0), ctypes.byref(rc),
                                       _ptr(amax), bits, _ptr(codes), ld, _ptr(s32), None,
                                       _ptr(sums), _stream(x)))
    return codes, s32, sums


def dequant(acc: torch.Tensor, scales: torch.Tensor, layer: PreparedLayer, *, out: str = "bf16",
            y: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The dequant loop of forward (pipeline.cpp:224-230) on int32
    accumulators summed outside K3 (row-parallel all-reduce)."""
    if acc.dtype != torch.int32 or acc.dim() != 2 or acc.stride(1) != 1:
        raise ShapeError("acc must be a row-major int32 matrix")
    M = acc.shape[0]
    if y is None:
        y = torch.empty((M, layer.out_features), dtype=_OUT_DTYPE[out], device=acc.device)
    else:
        _check_out(y, M, layer.out_features, out, layer.device)
    check(_lib().crt_dequant(_ptr(acc), acc.stride(0), M, _ptr(scales), layer.handle, _OUT[out],
                             _ptr(y), y.stride(0), _stream(acc)))
    return y


def quant_gemm_i8(codes: torch.Tensor, scales: torch.Tensor, sums: torch.Tensor,
                  layer: PreparedLayer, *, out: str = "bf16",
                  y: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K3 v3 (weights expanded in hardware by tcgen05.cp) on rotate_quantize_i8
    output."""
    M = codes.shape[0]
    N = layer.out_features
    if y is None:
        y = torch.empty((M, N), dtype=_OUT_DTYPE[out], device=codes.device)
    else:
        _check_out(y, M, N, out, layer.device)
    check(_lib().crt_quant_gemm_i8(_ptr(codes), codes.stride(0), _ptr(scales), _ptr(sums),
                                   layer.handle, M, _OUT[out], _ptr(y), y.stride(0),
                                   _stream(codes)))
    return y


def int_gemm(codes: torch.Tensor, layer: PreparedLayer, aq: QuantSpec = QuantSpec(4)):
    """Raw int32 accumulators (int_gemm, pipeline.cpp:178-204) of packed
    activation codes against the prepared weights."""
    ones = torch.ones(codes.shape[0], dtype=torch.float32, device=codes.device)
    return quant_gemm(codes, ones, layer, aq, out="i32")


def launch_count() -> int:
    """Kernels this library has launched so far (process lifetime)."""
    return int(_lib().crt_launch_count())
