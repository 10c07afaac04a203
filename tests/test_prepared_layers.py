"""f2: layers prepared and saved by the real reference
(tests/golden/prepared/, made by tests/golden/make_prepared.py) loaded onto
the GPU.  CPU: the CRT1 reader against the reference's files and its
format-error offsets (test_tensorio.cpp:82-131).  GPU: forward through the
loaded layer equals the reference's forward on that layer (int32
accumulators bit-exact, fp32 dequant within 1e-6 relative)."""
import os
import struct

import numpy as np
import pytest
import torch

from paper_2512_03673_b200._abi import FormatError
from paper_2512_03673_b200.tensorio import payload_bytes, read_tensor

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PREP = os.path.join(GOLD, "prepared")
CASES = sorted(os.listdir(PREP))


def test_reader_parses_reference_files():
    for case in CASES:
        d = os.path.join(PREP, case)
        meta = np.load(os.path.join(GOLD, "prepared.npz"))[f"{case}/meta"]
        m, k, n, kind, group, bits, has_bias = (int(v) for v in meta)
        w = read_tensor(os.path.join(d, "weights.crt"))
        assert w.dtype == ("packed_i4" if bits == 4 else "i8") and w.dims == [n, k]
        assert len(w.payload) == payload_bytes(w.dtype, w.dims)
        s = read_tensor(os.path.join(d, "weights.scales.crt"))
        assert s.dtype == "f32" and s.dims == [n]  # the reference saves f32 scales
        assert os.path.exists(os.path.join(d, "bias.crt")) == bool(has_bias)
        if bits == 4 and k % 2:  # odd rows pad with a zero nibble (tensorio.cpp:78-86)
            rows = np.frombuffer(w.payload, np.uint8).reshape(n, (k + 1) // 2)
            assert not (rows[:, -1] & 0xF0).any()


def _f32_2x2(path):
    hdr = b"CRT1" + bytes([0, 2]) + struct.pack("<QQ", 2, 2)
    open(path, "wb").write(hdr + np.arange(4, dtype=np.float32).tobytes())
    return open(path, "rb").read()


@pytest.mark.parametrize("mutate,offset", [
    (lambda b: b"X" + b[1:], 0),                 # bad magic
    (lambda b: b[:4] + bytes([9]) + b[5:], 4),   # unknown dtype
    (lambda b: b[:5] + bytes([0]) + b[6:], 5),   # ndim = 0
    (lambda b: b[:-3], None),                    # truncated payload -> offset = size
    (lambda b: b + b"\0", 38),                   # trailing bytes
])
def test_format_errors_carry_byte_offsets(tmp_path, mutate, offset):
    p = str(tmp_path / "x.crt")
    good = _f32_2x2(p)
    assert len(good) == 38  # test_tensorio.cpp:23 "2x2 file is 38 bytes"
    bad = mutate(good)
    open(p, "wb").write(bad)
    with pytest.raises(FormatError) as e:
        read_tensor(p)
    assert e.value.offset == (len(bad) if offset is None else offset)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_reference_prepared_layer_forward_on_gpu(case):
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import QuantSpec
    from paper_2512_03673_b200.tensorio import load_prepared_layer
    g = np.load(os.path.join(GOLD, "prepared.npz"))
    m, k, n, kind, group, bits, has_bias = (int(v) for v in g[f"{case}/meta"])
    layer = load_prepared_layer(os.path.join(PREP, case))
    assert (layer.out_features, layer.in_features) == (n, k)
    xb = g[f"{case}/x_bf16"]
    x = torch.from_numpy(xb.astype(np.uint16).view(np.int16)).cuda().view(torch.bfloat16)
    acc = crt.forward(x, layer, QuantSpec(bits), out="i32").cpu().numpy()
    assert np.array_equal(acc, g[f"{case}/acc"])
    y = crt.forward(x, layer, QuantSpec(bits), out="f32").cpu().numpy().astype(np.float64)
    want = g[f"{case}/values"]
    assert (np.abs(y - want) <= 1e-6 * np.abs(want) + 1e-6).all()
