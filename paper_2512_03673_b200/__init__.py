"""paper_2512_03673_b200 -- B200-native ConvLinear4bit forward path.

Drop-in for the reference's ConvRot / ConvLinear4bit hot path
(/root/reference/proj/core/src/pipeline.cpp:111-233): regular-Hadamard
group rotation + per-token INT4 quantize + nibble pack (K1), offline weight
preparation (K2) and the W4A4 tcgen05 GEMM with fused dequant (K3), all
hand-written for sm_100a behind the C-ABI in include/crt/convlinear4bit.h.
"""
from ._abi import (CapacityError, CudaError, Error, FormatError, InvalidOrderError,  # noqa: F401
                   InvalidValueError, ShapeError, UnsupportedError, load)
from .tensorio import load_prepared_layer, read_tensor  # noqa: F401
from .api import (PreparedLayer, QuantSpec, RotationKind, RotationSpec, Workspace,  # noqa: F401
                  dequant, forward, int_gemm, launch_count, packed_row_bytes, prepare_layer,
                  prepare_layer_kshard, prepare_layer_shard, quant_gemm, quant_gemm_i8, regular,
                  rotate_quantize, rotate_quantize_amax, rotate_quantize_i8,
                  rotate_quantize_into, sylvester)

__all__ = [
    "Error", "InvalidOrderError", "InvalidValueError", "ShapeError", "CapacityError",
    "FormatError", "CudaError", "UnsupportedError", "RotationKind", "RotationSpec", "QuantSpec",
    "PreparedLayer", "Workspace", "regular", "sylvester", "rotate_quantize", "rotate_quantize_into",
    "prepare_layer", "prepare_layer_shard", "prepare_layer_kshard", "forward", "quant_gemm",
    "quant_gemm_i8", "rotate_quantize_i8", "rotate_quantize_amax", "dequant", "int_gemm",
    "launch_count",
    "packed_row_bytes", "load", "load_prepared_layer", "read_tensor",
]
