"""Reference-prepared layers on the GPU.

Reads the reference's on-disk prepared layer -- ``save_prepared_layer``
(core/src/pipeline.cpp:257-314): ``weights.crt`` (packed_i4 or i8 codes),
``weights.scales.crt`` (f32!), optional ``bias.crt`` (f64) and
``manifest.json`` -- and uploads it through ``crt_layer_from_codes``.  The
CRT1 reader mirrors ``read_tensor`` (core/src/tensorio.cpp:94-128) including
its FormatError cases and byte offsets.  Host-side parsing only; the codes
are used on the device exactly as the reference saved them.
"""
from __future__ import annotations

import ctypes
import json
import os
import struct
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _abi
from ._abi import FormatError, check

MAGIC = b"CRT1"
DTYPES = {0: "f32", 1: "f64", 2: "i8", 3: "packed_i4"}  # tensorio.hpp:18


@dataclass
class Tensor:
    dtype: str
    dims: List[int]
    payload: bytes


def payload_bytes(dtype: str, dims: List[int]) -> int:
    """tensorio.cpp payload_bytes: packed_i4 rows padded to a whole byte."""
    n = 1
    for d in dims[:-1]:
        n *= d
    last = dims[-1]
    if dtype == "packed_i4":
        return n * ((last + 1) // 2)
    return n * last * {"f32": 4, "f64": 8, "i8": 1}[dtype]


def _format_error(what: str, offset: int) -> FormatError:
    e = FormatError(f"{what} (offset {offset})")
    e.offset = offset
    return e


def read_tensor(path: str) -> Tensor:
    """read_tensor (tensorio.cpp:94-128)."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise _format_error(f"cannot open file: {path}", 0) from None
    if len(data) < 6:
        raise _format_error("truncated header", len(data))
    if data[:4] != MAGIC:
        raise _format_error("bad magic", 0)
    if data[4] not in DTYPES:
        raise _format_error(f"unknown dtype {data[4]}", 4)
    dtype, ndim = DTYPES[data[4]], data[5]
    if ndim == 0:
        raise _format_error("ndim must be >= 1", 5)
    off = 6
    if len(data) < off + 8 * ndim:
        raise _format_error("truncated dims", len(data))
    dims = list(struct.unpack_from("<" + "Q" * ndim, data, off))
    off += 8 * ndim
    expected = payload_bytes(dtype, dims)
    if len(data) - off < expected:
        raise _format_error("truncated payload", len(data))
    if len(data) - off > expected:
        raise _format_error("trailing bytes after payload", off + expected)
    return Tensor(dtype, dims, data[off:])


def _vector(t: Tensor) -> np.ndarray:
    """vector_from_tensor: f32 / f64, 1-D."""
    if len(t.dims) != 1 or t.dtype not in ("f32", "f64"):
        raise _format_error("expected a 1-D f32/f64 tensor", 4)
    return np.frombuffer(t.payload, dtype=np.float32 if t.dtype == "f32" else np.float64)


def load_prepared_layer(path: str, device=None):
    """load_prepared_layer (pipeline.cpp:288-314) straight onto the GPU:
    returns an api.PreparedLayer whose codes / scales / bias are the files'."""
    import torch

    from . import api
    try:
        manifest = json.load(open(os.path.join(path, "manifest.json")))
    except OSError:
        raise _format_error(f"missing manifest.json in {path}", 0) from None
    n, k, bits = int(manifest["out_features"]), int(manifest["in_features"]), int(manifest["bits"])
    rot = manifest["rotation"]
    kind = {"none": api.RotationKind.none, "sylvester": api.RotationKind.sylvester,
            "regular": api.RotationKind.regular}.get(rot["kind"])
    if kind is None:
        raise api.UnsupportedError(f"rotation kind {rot['kind']} is not built here")
    spec = api.RotationSpec(kind, int(rot["group_size"]), int(rot["seed"]),
                            bool(rot["identity_tail"]))
    w = read_tensor(os.path.join(path, "weights.crt"))
    want = "packed_i4" if bits == 4 else "i8"
    if w.dtype != want or w.dims != [n, k]:
        raise _format_error(f"weights.crt: expected {want} [{n}, {k}]", 4)
    scales = np.ascontiguousarray(_vector(read_tensor(os.path.join(path, "weights.scales.crt"))),
                                  dtype=np.float32)
    if scales.shape[0] != n:
        raise _format_error("weights.scales.crt length != out_features", 6)
    bias = None
    bpath = os.path.join(path, "bias.crt")
    if os.path.exists(bpath):
        bias = np.ascontiguousarray(_vector(read_tensor(bpath)), dtype=np.float64)
        if bias.shape[0] != n:
            raise _format_error("bias.crt length != out_features", 6)
    codes = np.frombuffer(w.payload, dtype=np.uint8)
    ld = (k + 1) // 2 if bits == 4 else k
    dev = torch.device(device) if device is not None else torch.device("cuda")
    desc = _abi.LayerDescC(n, k, spec.c(), bits, _abi.CRT_DTYPE_BF16)
    h = ctypes.c_void_p()
    with torch.cuda.device(dev):
        st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        check(_abi.load().crt_layer_from_codes(
            ctypes.byref(desc), codes.ctypes.data_as(ctypes.c_void_p), ld,
            scales.ctypes.data_as(ctypes.c_void_p),
            None if bias is None else bias.ctypes.data_as(ctypes.c_void_p), st, ctypes.byref(h)))
    return api.PreparedLayer(h.value, n, k, spec, api.QuantSpec(bits), bias is not None,
                             str(manifest.get("name", "")), dev)
