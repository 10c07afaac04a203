"""TEST INFRASTRUCTURE ONLY -- the parity checker.

ctypes/numpy front end for
  * ``oracle/_build/liboracle.so``: the plain-C restatement of the reference
    CPU path (``oracle/convrot_oracle.c``; every function cites the reference
    file:line it restates), and
  * ``oracle/_ref/libconvrot_ref.so``: the UNMODIFIED reference core compiled
    in place from /root/reference by ``oracle/Makefile`` (absent on boxes that
    never saw /root/reference unless the prebuilt file travelled with the
    repo snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2512_03673_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libconvrot_ref.so")

ROT_NONE, ROT_SYLVESTER, ROT_REGULAR = 0, 1, 2
MODE_ROWWISE, MODE_COLWISE, MODE_GAUSSIAN = 0, 1, 2

STATUS_NAMES = {0: "OK", 1: "INVALID_ORDER", 2: "INVALID_VALUE", 3: "SHAPE",
                4: "CAPACITY", 5: "FORMAT"}


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {what}")


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_U64 = ctypes.c_uint64

_lib: Optional[ctypes.CDLL] = None
_ref: Optional[ctypes.CDLL] = None


def build(ref: bool = False) -> None:
    """Build the C restatement (and the reference core when asked and its
    sources are present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        sig = {
            "or_regular": (_I, [_I, _P]),
            "or_sylvester": (_I, [_I, _P]),
            "or_group_rotate": (_I, [_P, _I64, _I64, _I, _I, _I, _P]),
            "or_compute_scales": (_I, [_P, _I64, _I64, _I, _P]),
            "or_quantize": (_I, [_P, _I64, _I64, _P, _I, _P]),
            "or_pack_int4": (_I, [_P, _I64, _P]),
            "or_unpack_int4": (None, [_P, _I64, _P]),
            "or_pack_int4_rows": (_I, [_P, _I64, _I64, _P]),
            "or_int_gemm": (_I, [_P, _P, _I64, _I64, _I64, _I, _I, _P]),
            "or_int_gemm_check": (_I, [_I64, _I, _I]),
            "or_dequant": (None, [_P, _I64, _I64, _P, _P, _P, _P]),
            "or_prepare_layer": (_I, [_P, _I64, _I64, _I, _I, _I, _I, _P, _P]),
            "or_forward": (_I, [_P, _I64, _I64, _P, _P, _P, _I64, _I, _I, _I, _I,
                                _I, _P, _P, _P, _P]),
            "or_reference_forward": (_I, [_P, _P, _P, _I64, _I64, _I64, _P]),
            "or_gaussian_matrix": (None, [_I64, _I64, _U64, _P]),
            "or_rng_u64": (None, [_U64, _I64, _P]),
            "or_synth_outliers": (_I, [_I64, _I64, _I, _D, _D, _U64, _P]),
            "or_to_bf16": (None, [_P, _I64, _P]),
            "or_from_bf16": (None, [_P, _I64, _P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> ctypes.CDLL:
    """The real reference core (oracle/_ref).  Raises if it was never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = ctypes.CDLL(REF_SO)
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_thread_count": (ctypes.c_uint, []),
            "ref_regular": (_I, [_I, _P]),
            "ref_group_rotate": (_I, [_P, _I64, _I64, _I, _I, _I, _P]),
            "ref_compute_scales": (_I, [_P, _I64, _I64, _I, _P]),
            "ref_quantize": (_I, [_P, _I64, _I64, _P, _I, _P]),
            "ref_pack_rows": (_I, [_P, _I64, _I64, _P]),
            "ref_int_gemm": (_I, [_P, _P, _I64, _I64, _I64, _I, _I, _P]),
            "ref_prepare_layer": (_I, [_P, _I64, _I64, _P, _I, _I, _I, _I, _P, _P]),
            "ref_forward": (_I, [_P, _I64, _I64, _P, _I64, _P, _I, _I, _I, _I, _I,
                                 _P, _P, _P, _P]),
            "ref_forward_prepared": (_I, [_P, _I64, _I64, _P, _P, _P, _I64, _I, _I,
                                          _I, _I, _I, _P]),
            "ref_reference_forward": (_I, [_P, _P, _P, _I64, _I64, _I64, _P]),
            "ref_synth_outliers": (_I, [_I64, _I64, _I, _D, _D, _U64, _P]),
            "ref_gaussian_matrix": (None, [_I64, _I64, _U64, _P]),
            "ref_rng_u64": (None, [_U64, _I64, _P]),
            "ref_save_prepared_layer": (_I, [ctypes.c_char_p, _P, _I64, _I64, _P, _I,
                                             _I, _I, _I]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _ref = L
    return _ref


# --------------------------------------------------------------------------
# numpy helpers
# --------------------------------------------------------------------------
def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(st: int, who: str = "oracle") -> None:
    if st != 0:
        what = ""
        if who == "ref":
            what = ref().ref_last_error().decode()
        raise OracleError(st, what)


def regular(n: int) -> np.ndarray:
    """regular(n) sign matrix (hadamard.cpp:91-106) as int8 n x n."""
    out = np.empty((n, n), np.int8) if n > 0 and n <= 4096 else np.empty((1,), np.int8)
    _check(lib().or_regular(n, _p(out)))
    return out


def sylvester(n: int) -> np.ndarray:
    out = np.empty((n, n), np.int8) if n > 0 and n <= 4096 else np.empty((1,), np.int8)
    _check(lib().or_sylvester(n, _p(out)))
    return out


def group_rotate(x, kind: int = ROT_REGULAR, group: int = 16,
                 identity_tail: bool = False) -> np.ndarray:
    x = _f64(x)
    out = np.empty_like(x)
    _check(lib().or_group_rotate(_p(x), x.shape[0], x.shape[1], kind, group,
                                 int(identity_tail), _p(out)))
    return out


def compute_scales(x, bits: int = 4) -> np.ndarray:
    x = _f64(x)
    s = np.empty(x.shape[0], np.float64)
    _check(lib().or_compute_scales(_p(x), x.shape[0], x.shape[1], bits, _p(s)))
    return s


def quantize(x, scales, bits: int = 4) -> np.ndarray:
    x = _f64(x)
    s = _f64(scales)
    c = np.empty(x.shape, np.int8)
    _check(lib().or_quantize(_p(x), x.shape[0], x.shape[1], _p(s), bits, _p(c)))
    return c


def pack_int4_rows(codes) -> np.ndarray:
    c = np.ascontiguousarray(codes, dtype=np.int8)
    rows, cols = c.shape
    out = np.empty((rows, (cols + 1) // 2), np.uint8)
    _check(lib().or_pack_int4_rows(_p(c), rows, cols, _p(out)))
    return out


def unpack_int4_rows(packed, cols: int) -> np.ndarray:
    p = np.ascontiguousarray(packed, dtype=np.uint8)
    rows = p.shape[0]
    out = np.empty((rows, cols), np.int8)
    for i in range(rows):
        lib().or_unpack_int4(_p(p[i]), cols, _p(out[i]))
    return out


def unpack_int4_rows_np(packed, cols: int) -> np.ndarray:
    """Vectorised unpack (same semantics as quant.cpp:83-96)."""
    p = np.ascontiguousarray(packed, dtype=np.uint8)
    lo = (p & 0x0F).astype(np.int8)
    hi = (p >> 4).astype(np.int8)
    lo = np.where(lo >= 8, lo - 16, lo).astype(np.int8)
    hi = np.where(hi >= 8, hi - 16, hi).astype(np.int8)
    out = np.empty((p.shape[0], p.shape[1] * 2), np.int8)
    out[:, 0::2] = lo
    out[:, 1::2] = hi
    return out[:, :cols]


def int_gemm(a, b, bits_a: int = 4, bits_b: int = 4) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int8)
    b = np.ascontiguousarray(b, dtype=np.int8)
    if a.shape[1] != b.shape[1]:
        raise OracleError(3, "int_gemm: inner dimensions differ")
    out = np.empty((a.shape[0], b.shape[0]), np.int32)
    _check(lib().or_int_gemm(_p(a), _p(b), a.shape[0], b.shape[0], a.shape[1],
                             bits_a, bits_b, _p(out)))
    return out


def dequant(acc, s_a, s_w, bias=None) -> np.ndarray:
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    s_a, s_w = _f64(s_a), _f64(s_w)
    b = None if bias is None else _f64(bias)
    out = np.empty(acc.shape, np.float64)
    lib().or_dequant(_p(acc), acc.shape[0], acc.shape[1], _p(s_a), _p(s_w), _p(b),
                     _p(out))
    return out


def prepare_layer(w, kind: int = ROT_REGULAR, group: int = 16,
                  identity_tail: bool = False, bits: int = 4):
    """(codes int8 N x K, scales f64 N) as prepare_layer (pipeline.cpp:158-176)."""
    w = _f64(w)
    n, k = w.shape
    codes = np.empty((n, k), np.int8)
    scales = np.empty(n, np.float64)
    _check(lib().or_prepare_layer(_p(w), n, k, kind, group, int(identity_tail), bits,
                                  _p(codes), _p(scales)))
    return codes, scales


def forward(x, w_codes, w_scales, bias=None, kind: int = ROT_REGULAR, group: int = 16,
            identity_tail: bool = False, bits_a: int = 4, bits_w: int = 4):
    """forward (pipeline.cpp:206-233).  Returns dict(values, act_codes,
    act_scales, acc)."""
    x = _f64(x)
    m, k = x.shape
    wc = np.ascontiguousarray(w_codes, dtype=np.int8)
    n = wc.shape[0]
    if wc.shape[1] != k:
        raise OracleError(3, "forward: shape mismatch")
    ws = _f64(w_scales)
    b = None if bias is None else _f64(bias)
    out = np.empty((m, n), np.float64)
    codes = np.empty((m, k), np.int8)
    sa = np.empty(m, np.float64)
    acc = np.empty((m, n), np.int32)
    _check(lib().or_forward(_p(x), m, k, _p(wc), _p(ws), _p(b), n, kind, group,
                            int(identity_tail), bits_a, bits_w, _p(out), _p(codes),
                            _p(sa), _p(acc)))
    return {"values": out, "act_codes": codes, "act_scales": sa, "acc": acc}


def reference_forward(x, w, bias=None) -> np.ndarray:
    x, w = _f64(x), _f64(w)
    b = None if bias is None else _f64(bias)
    out = np.empty((x.shape[0], w.shape[0]), np.float64)
    _check(lib().or_reference_forward(_p(x), _p(w), _p(b), x.shape[0], w.shape[0],
                                      x.shape[1], _p(out)))
    return out


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty((rows, cols), np.float64)
    lib().or_gaussian_matrix(rows, cols, seed, _p(out))
    return out


def rng_u64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().or_rng_u64(seed, n, _p(out))
    return out


def synth_outliers(rows: int, cols: int, mode: int, magnitude: float, fraction: float,
                   seed: int) -> np.ndarray:
    out = np.empty((rows, cols), np.float64)
    _check(lib().or_synth_outliers(rows, cols, mode, magnitude, fraction, seed, _p(out)))
    return out


def to_bf16_bits(x) -> np.ndarray:
    """double -> f32 (RNE) -> bf16 (RNE), the torch narrowing path."""
    x = _f64(x)
    out = np.empty(x.shape, np.uint16)
    lib().or_to_bf16(_p(x), x.size, _p(out))
    return out


def from_bf16_bits(b) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.uint16)
    out = np.empty(b.shape, np.float64)
    lib().or_from_bf16(_p(b), b.size, _p(out))
    return out


def synth_input(rows: int, cols: int, family: str, seed: int) -> np.ndarray:
    """The harness input families: ``gaussian``;
    ``colwise`` c=50 f=0.01; ``rowwise`` c=100 f=0.05 -- drawn with the
    pinned RNG, narrowed to bf16.  Returns bf16 bit patterns (uint16)."""
    if family == "gaussian":
        x = synth_outliers(rows, cols, MODE_GAUSSIAN, 1.0, 1.0, seed)
    elif family == "colwise":
        x = synth_outliers(rows, cols, MODE_COLWISE, 50.0, 0.01, seed)
    elif family == "rowwise":
        x = synth_outliers(rows, cols, MODE_ROWWISE, 100.0, 0.05, seed)
    else:
        raise ValueError(family)
    return to_bf16_bits(x)


# --------------------------------------------------------------------------
# the real reference (oracle/_ref)
# --------------------------------------------------------------------------
class Ref:
    """Calls into the unmodified reference core."""

    @staticmethod
    def regular(n: int) -> np.ndarray:
        out = np.empty((n, n), np.int8) if 0 < n <= 4096 else np.empty((1,), np.int8)
        _check(ref().ref_regular(n, _p(out)), "ref")
        return out

    @staticmethod
    def group_rotate(x, kind=ROT_REGULAR, group=16, identity_tail=False):
        x = _f64(x)
        out = np.empty_like(x)
        _check(ref().ref_group_rotate(_p(x), x.shape[0], x.shape[1], kind, group,
                                      int(identity_tail), _p(out)), "ref")
        return out

    @staticmethod
    def compute_scales(x, bits=4):
        x = _f64(x)
        s = np.empty(x.shape[0], np.float64)
        _check(ref().ref_compute_scales(_p(x), x.shape[0], x.shape[1], bits, _p(s)), "ref")
        return s

    @staticmethod
    def quantize(x, scales, bits=4):
        x = _f64(x)
        s = _f64(scales)
        c = np.empty(x.shape, np.int8)
        _check(ref().ref_quantize(_p(x), x.shape[0], x.shape[1], _p(s), bits, _p(c)), "ref")
        return c

    @staticmethod
    def pack_rows(codes):
        c = np.ascontiguousarray(codes, dtype=np.int8)
        out = np.empty((c.shape[0], (c.shape[1] + 1) // 2), np.uint8)
        _check(ref().ref_pack_rows(_p(c), c.shape[0], c.shape[1], _p(out)), "ref")
        return out

    @staticmethod
    def int_gemm(a, b, bits_a=4, bits_b=4):
        a = np.ascontiguousarray(a, dtype=np.int8)
        b = np.ascontiguousarray(b, dtype=np.int8)
        out = np.empty((a.shape[0], b.shape[0]), np.int32)
        _check(ref().ref_int_gemm(_p(a), _p(b), a.shape[0], b.shape[0], a.shape[1],
                                  bits_a, bits_b, _p(out)), "ref")
        return out

    @staticmethod
    def prepare_layer(w, bias=None, kind=ROT_REGULAR, group=16, identity_tail=False,
                      bits=4):
        w = _f64(w)
        n, k = w.shape
        b = None if bias is None else _f64(bias)
        codes = np.empty((n, k), np.int8)
        scales = np.empty(n, np.float64)
        _check(ref().ref_prepare_layer(_p(w), n, k, _p(b), kind, group,
                                       int(identity_tail), bits, _p(codes),
                                       _p(scales)), "ref")
        return codes, scales

    @staticmethod
    def forward(x, w, bias=None, kind=ROT_REGULAR, group=16, identity_tail=False,
                bits_a=4, bits_w=4, internals=True):
        x, w = _f64(x), _f64(w)
        m, k = x.shape
        n = w.shape[0]
        b = None if bias is None else _f64(bias)
        out = np.empty((m, n), np.float64)
        codes = np.empty((m, k), np.int8) if internals else None
        sa = np.empty(m, np.float64) if internals else None
        acc = np.empty((m, n), np.int32) if internals else None
        _check(ref().ref_forward(_p(x), m, k, _p(w), n, _p(b), kind, group,
                                 int(identity_tail), bits_a, bits_w, _p(out), _p(codes),
                                 _p(sa), _p(acc)), "ref")
        return {"values": out, "act_codes": codes, "act_scales": sa, "acc": acc}

    @staticmethod
    def forward_prepared(x, w_codes, w_scales, bias=None, kind=ROT_REGULAR, group=16,
                         identity_tail=False, bits_a=4, bits_w=4):
        x = _f64(x)
        m, k = x.shape
        wc = np.ascontiguousarray(w_codes, dtype=np.int8)
        n = wc.shape[0]
        ws = _f64(w_scales)
        b = None if bias is None else _f64(bias)
        out = np.empty((m, n), np.float64)
        _check(ref().ref_forward_prepared(_p(x), m, k, _p(wc), _p(ws), _p(b), n, kind,
                                          group, int(identity_tail), bits_a, bits_w,
                                          _p(out)), "ref")
        return out

    @staticmethod
    def save_prepared_layer(path, w, bias=None, kind=ROT_REGULAR, group=16,
                            identity_tail=False, bits=4):
        """The reference's prepare_layer + save_prepared_layer
        (pipeline.cpp:158-176, :257-287) into directory `path`."""
        w = _f64(w)
        n, k = w.shape
        b = None if bias is None else _f64(bias)
        _check(ref().ref_save_prepared_layer(path.encode(), _p(w), n, k, _p(b), kind, group,
                                             int(identity_tail), bits), "ref")

    @staticmethod
    def reference_forward(x, w, bias=None):
        x, w = _f64(x), _f64(w)
        b = None if bias is None else _f64(bias)
        out = np.empty((x.shape[0], w.shape[0]), np.float64)
        _check(ref().ref_reference_forward(_p(x), _p(w), _p(b), x.shape[0], w.shape[0],
                                           x.shape[1], _p(out)), "ref")
        return out

    @staticmethod
    def synth_outliers(rows, cols, mode, magnitude, fraction, seed):
        out = np.empty((rows, cols), np.float64)
        _check(ref().ref_synth_outliers(rows, cols, mode, magnitude, fraction, seed,
                                        _p(out)), "ref")
        return out

    @staticmethod
    def gaussian_matrix(rows, cols, seed):
        out = np.empty((rows, cols), np.float64)
        ref().ref_gaussian_matrix(rows, cols, seed, _p(out))
        return out

    @staticmethod
    def rng_u64(seed, n):
        out = np.empty(n, np.uint64)
        ref().ref_rng_u64(seed, n, _p(out))
        return out


def rel_frobenius_error(got, want) -> float:
    """test_util.hpp:58-66."""
    import math
    got, want = _f64(got).ravel(), _f64(want).ravel()
    err = 0.0
    for g, w in zip(got.tolist(), want.tolist()):  # sequential, like the C++
        d = g - w
        err += d * d
    total = 0.0
    for w in want.tolist():
        total += w * w
    refn = math.sqrt(total)
    return math.sqrt(err) if refn == 0.0 else math.sqrt(err) / refn
