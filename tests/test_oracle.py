"""The oracle (plain-C restatement, oracle/convrot_oracle.c) pinned against
the reference's own known answers and against golden vectors made by the
real reference (tests/golden/make_golden.py).  CPU only."""
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


# --- known answers copied from the reference's own tests -------------------
def test_h4_literal_and_sign_text():
    # test_hadamard.cpp:75-84, :233-236
    h = O.regular(4)
    text = "".join("".join("+" if v > 0 else "-" for v in row) + "\n" for row in h)
    assert text == "+++-\n++-+\n+-++\n-+++\n"


@pytest.mark.parametrize("n", [4, 16, 64, 256])
def test_regular_row_and_column_sums(n):
    # hadamard.hpp:46-48: all row/column sums equal +sqrt(n); test_hadamard.cpp:86-90
    h = O.regular(n).astype(np.int64)
    assert (h.sum(0) == int(np.sqrt(n))).all() and (h.sum(1) == int(np.sqrt(n))).all()
    assert (h @ h.T == n * np.eye(n, dtype=np.int64)).all()
    assert (h == h.T).all()


def test_regular_discrepancy():
    # test_hadamard.cpp:142-150: discrepancy 2 / 8 for n = 4 / 64
    assert np.abs(O.regular(4).astype(int).sum(0)).max() == 2
    assert np.abs(O.regular(64).astype(int).sum(0)).max() == 8


@pytest.mark.parametrize("n", [0, 2, 8, 12, 32, 8192, 16384])
def test_regular_rejects_bad_orders(n):
    # hadamard.cpp:92-96 (test_hadamard.cpp:106-111)
    with pytest.raises(O.OracleError) as e:
        O.regular(n)
    assert e.value.status == 1


def test_kronecker_digit_rule():
    # hadamard.cpp:119: right factor on the least-significant base-4 digit
    h16 = O.regular(16)
    h4 = O.regular(4)
    for r in range(16):
        for c in range(16):
            assert h16[r, c] == h4[r // 4, c // 4] * h4[r % 4, c % 4]


def test_half_even_examples():
    # test_quant.cpp:32-45
    x = np.array([[0.5, -3.5, 7.0]])
    assert O.quantize(x, [1.0]).tolist() == [[0, -4, 7]]
    row = np.array([[1.0, 2, 3, 4]])
    s = O.compute_scales(row)
    assert s[0] == 4.0 / 7.0
    assert O.quantize(row, s).tolist() == [[2, 4, 5, 7]]


def test_scales_zero_row_and_nonfinite():
    # test_quant.cpp:12-30
    x = np.array([[0.5, -3.5, 7.0], [0, 0, 0], [1.0, 2.0, 4.0]])
    s = O.compute_scales(x)
    assert s.tolist() == [1.0, 1.0, 4.0 / 7.0]
    for bad in (np.nan, np.inf):
        with pytest.raises(O.OracleError) as e:
            O.compute_scales(np.array([[1.0, bad]]))
        assert e.value.status == 2


def test_pack_bytes():
    # test_quant.cpp:122-138
    assert O.pack_int4_rows(np.array([[-7, 7]], np.int8)).tolist() == [[0x79]]
    assert O.pack_int4_rows(np.array([[5, -3, -8]], np.int8)).tolist() == [[0xD5, 0x08]]
    with pytest.raises(O.OracleError):
        O.pack_int4_rows(np.array([[9]], np.int8))


def test_pinned_seeded_golden_bit_exact():
    # test_pipeline.cpp:182-193 pins 0.12035518741210707 (epsilon 0.1); the
    # restatement reproduces it to the last bit.
    x = O.gaussian_matrix(16, 64, 15)
    w = O.gaussian_matrix(8, 64, 515)
    wc, ws = O.prepare_layer(w, O.ROT_REGULAR, 16)
    f = O.forward(x, wc, ws, None, O.ROT_REGULAR, 16)
    err = O.rel_frobenius_error(f["values"], O.reference_forward(x, w))
    assert err == 0.12035518741210707


def test_rng_amplitude_pins():
    # test_analysis.cpp:42-56
    assert np.abs(O.gaussian_matrix(100, 100, 42)).max() == 4.207415109866564
    assert np.abs(O.synth_outliers(32, 64, O.MODE_ROWWISE, 100, 0.05, 7)).max() == 279.65078105838967
    assert np.abs(O.synth_outliers(16, 32, O.MODE_COLWISE, 50, 0.1, 9)).max() == 137.23812707653872


def test_one_by_one_and_zero_activations():
    # test_pipeline.cpp:154-180
    wc, ws = O.prepare_layer(np.array([[7.0]]), O.ROT_NONE, 0)
    assert O.forward(np.array([[7.0]]), wc, ws, None, O.ROT_NONE, 0)["values"].tolist() == [[49.0]]
    w = O.gaussian_matrix(3, 4, 9)
    wc, ws = O.prepare_layer(w, O.ROT_NONE, 0)
    bias = np.array([0.5, -1.5, 2.0])
    out = O.forward(np.zeros((2, 4)), wc, ws, bias, O.ROT_NONE, 0)["values"]
    assert (out == bias[None, :]).all()


def test_integer_grid_forward_is_exact():
    # test_pipeline.cpp:219-227
    x = np.array([[7, -3, 0, 2], [1, -7, 5, 4]], np.float64)
    w = np.array([[7, 1, -1, 0], [-2, 7, 3, 1], [0, -5, 7, -6]], np.float64)
    wc, ws = O.prepare_layer(w, O.ROT_NONE, 0)
    got = O.forward(x, wc, ws, None, O.ROT_NONE, 0)["values"]
    assert (got == O.reference_forward(x, w)).all()


def test_int_gemm_capacity():
    # test_pipeline.cpp:144-152 / pipeline.cpp:184-192
    assert lib_check(200000, 8, 8) == 4
    assert lib_check(200000, 4, 4) == 0
    assert lib_check(43826196, 4, 4) == 0
    assert lib_check(43826197, 4, 4) == 4


def lib_check(k, a, b):
    return O.lib().or_int_gemm_check(k, a, b)


def test_group_order_and_divisibility():
    # test_pipeline.cpp:56-83
    x = O.gaussian_matrix(2, 10, 3)
    with pytest.raises(O.OracleError) as e:
        O.group_rotate(x, O.ROT_REGULAR, 4)
    assert e.value.status == 3
    out = O.group_rotate(x, O.ROT_REGULAR, 4, identity_tail=True)
    assert (out[:, 8:] == x[:, 8:]).all()
    with pytest.raises(O.OracleError) as e:
        O.group_rotate(O.gaussian_matrix(2, 16, 6), O.ROT_REGULAR, 8)
    assert e.value.status == 1


# --- golden vectors from the real reference --------------------------------
def _cases():
    g = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in g.files})
    return g, names


@pytest.mark.parametrize("name", _cases()[1])
def test_oracle_matches_reference_golden(name):
    g, _ = _cases()
    d = {k.split("/")[1]: g[k] for k in g.files if k.startswith(name + "/")}
    kind, group, tail, bits_a, bits_w, has_bias = d["meta"].tolist()
    x = O.from_bf16_bits(d["x_bf16"])
    w = O.from_bf16_bits(d["w_bf16"])
    bias = d["bias"] if has_bias else None
    wc, ws = O.prepare_layer(w, kind, group, bool(tail), bits_w)
    assert np.array_equal(wc, d["w_codes"])
    assert np.array_equal(ws, d["w_scales"])
    f = O.forward(x, wc, ws, bias, kind, group, bool(tail), bits_a, bits_w)
    assert np.array_equal(f["act_codes"], d["act_codes"])
    assert np.array_equal(f["act_scales"], d["act_scales"])
    assert np.array_equal(f["acc"], d["acc"])
    assert np.array_equal(f["values"], d["values"])
    assert np.array_equal(O.reference_forward(x, w, bias), d["ref_values"])
    if bits_a == 4:
        assert np.array_equal(O.pack_int4_rows(f["act_codes"]), d["act_packed"])
        assert np.array_equal(O.unpack_int4_rows_np(d["act_packed"], x.shape[1]),
                              d["act_codes"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_restatement_matches_reference_on_fresh_inputs():
    for n0 in (4, 16, 64, 256):
        xb = O.synth_input(9, 768, "colwise", 100 + n0)
        x = O.from_bf16_bits(xb)
        a = O.group_rotate(x, O.ROT_REGULAR, n0)
        b = O.Ref.group_rotate(x, O.ROT_REGULAR, n0)
        assert np.array_equal(a, b)
        sa, sb = O.compute_scales(a), O.Ref.compute_scales(b)
        assert np.array_equal(sa, sb)
        assert np.array_equal(O.quantize(a, sa), O.Ref.quantize(b, sb))
