"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/crt/convlinear4bit.h declares, host-only entry points match
the oracle, and shape/order/capacity errors are reported synchronously with
the reference's taxonomy -- all without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import _abi

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "crt",
                      "convlinear4bit.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(crt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_abi.EXPORTED)


def test_abi_version():
    assert _abi.load().crt_abi_version() == 1


@pytest.mark.parametrize("n", [4, 16, 64, 256, 1024])
def test_regular_matches_oracle(n):
    assert np.array_equal(crt.regular(n), O.regular(n))


@pytest.mark.parametrize("n", [2, 8, 64, 512])
def test_sylvester_matches_oracle(n):
    assert np.array_equal(crt.sylvester(n), O.sylvester(n))


@pytest.mark.parametrize("n", [0, 2, 8, 32, 8192, -4])
def test_regular_rejects_bad_orders(n):
    with pytest.raises(crt.InvalidOrderError):
        crt.regular(n)


def _rq(kind, group, k, tail=0, bits=4):
    lib = _abi.load()
    spec = _abi.RotationSpecC(kind, group, 0, tail)
    # host-side validation happens before any device pointer is touched
    return lib.crt_rotate_quant(ctypes.c_void_p(16), 0, 2, k, k, ctypes.byref(spec), bits,
                                ctypes.c_void_p(16), 4096, None, None, None)


def test_rotation_validation_mirrors_group_rotate():
    # pipeline.cpp:27-50, :111-130 (test_pipeline.cpp:56-83)
    assert _rq(2, 8, 16) == _abi.CRT_ERR_INVALID_ORDER      # regular needs 4^k
    assert _rq(2, 4, 10) == _abi.CRT_ERR_SHAPE              # not divisible
    assert _rq(2, 0, 12) == _abi.CRT_ERR_INVALID_ORDER      # global 12 not 4^k
    assert _rq(1, 0, 12) == _abi.CRT_ERR_INVALID_ORDER      # sylvester global 12
    assert _rq(2, -4, 16) == _abi.CRT_ERR_INVALID_VALUE     # negative group
    assert _rq(2, 16, 16, bits=5) == _abi.CRT_ERR_INVALID_VALUE
    assert _rq(2, 8192, 8192) == _abi.CRT_ERR_INVALID_ORDER  # > 4096


def test_capacity_precheck_is_host_side():
    # pipeline.cpp:184-192: int8 x int8 at K = 200,000 must be rejected.
    lib = _abi.load()
    assert O.lib().or_int_gemm_check(200000, 8, 8) == 4
    # no layer -> INVALID_VALUE before anything else; the capacity rule itself
    # is exercised on the GPU path (tests/test_gpu_parity.py).
    assert lib.crt_quant_gemm(None, 0, None, 4, None, 1, 0, None, 0, None) == \
        _abi.CRT_ERR_INVALID_VALUE


def test_error_classes_follow_reference_taxonomy():
    assert issubclass(crt.InvalidOrderError, crt.Error)
    assert issubclass(crt.ShapeError, crt.Error)
    assert crt.CapacityError.status == 4 and crt.FormatError.status == 5
