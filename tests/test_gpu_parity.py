"""GPU parity of the sm_100a path against the oracle (CPU restatement of the
reference) and the golden vectors made by the real reference.

Bars:
  * K1/K2 codes (packed bytes) and fp64 scales: bit-exact.
  * int32 accumulators: bit-exact.
  * fp32 dequant output: |y - ref| <= 1e-6 * (|acc*s_a*s_w| + |b|) + 1e-30
    (well inside the 1e-3 relative the north star asks).
  * bf16 output: within bf16 rounding (2^-8 relative) of the fp32 value.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")
DEV = "cuda"


def bf16_tensor(bits: np.ndarray) -> torch.Tensor:
    t = torch.from_numpy(bits.astype(np.uint16).view(np.int16)).to(DEV)
    return t.view(torch.bfloat16)


def kind_of(k):
    return {O.ROT_NONE: RotationKind.none, O.ROT_SYLVESTER: RotationKind.sylvester,
            O.ROT_REGULAR: RotationKind.regular}[k]


def golden_cases():
    g = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in g.files})
    return names


def load_case(name):
    g = np.load(GOLDEN)
    return {k.split("/")[1]: g[k] for k in g.files if k.startswith(name + "/")}


def check_dequant(y32, acc, sa, sw, bias):
    base = acc.astype(np.float64) * sa[:, None] * sw[None, :]
    ref = base + (bias[None, :] if bias is not None else 0.0)
    tol = 1e-6 * (np.abs(base) + (np.abs(bias)[None, :] if bias is not None else 0.0)) + 1e-30
    err = np.abs(y32.astype(np.float64) - ref)
    assert (err <= tol).all(), float((err / np.maximum(tol, 1e-300)).max())


# ---------------------------------------------------------------------------
# golden vectors from the real reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", golden_cases())
def test_golden_k1_k2_k3(name):
    d = load_case(name)
    kind, group, tail, bits_a, bits_w, has_bias = d["meta"].tolist()
    spec = RotationSpec(kind_of(kind), group, 0, bool(tail))
    x = bf16_tensor(d["x_bf16"])
    w = bf16_tensor(d["w_bf16"])
    M, K = x.shape
    N = w.shape[0]
    # K1
    codes, s32, s64 = crt.rotate_quantize(x, spec, QuantSpec(bits_a), scales64=True)
    row = crt.packed_row_bytes(K, bits_a)
    got = codes[:, :row].cpu().numpy()
    want = d["act_packed"] if bits_a == 4 else d["act_codes"].view(np.uint8)
    assert np.array_equal(got, want)
    assert np.array_equal(s64.cpu().numpy(), d["act_scales"])
    assert np.array_equal(s32.cpu().numpy(), d["act_scales"].astype(np.float32))
    # K2
    bias = torch.from_numpy(d["bias"].astype(np.float32)).to(DEV) if has_bias else None
    layer = crt.prepare_layer(w, bias, spec, QuantSpec(bits_w))
    wc, ws32, ws64 = layer.export()
    wwant = d["w_packed"] if bits_w == 4 else d["w_codes"].view(np.uint8)
    assert np.array_equal(wc.cpu().numpy(), wwant)
    assert np.array_equal(ws64.cpu().numpy(), d["w_scales"])
    # K3: accumulators, fp32 dequant, bf16
    acc = crt.forward(x, layer, QuantSpec(bits_a), out="i32")
    assert np.array_equal(acc.cpu().numpy(), d["acc"])
    y32 = crt.forward(x, layer, QuantSpec(bits_a), out="f32").cpu().numpy()
    check_dequant(y32, d["acc"], d["act_scales"], d["w_scales"], d["bias"] if has_bias else None)
    rel = np.abs(y32 - d["values"]) / np.maximum(np.abs(d["values"]), 1e-6)
    assert (np.abs(y32 - d["values"]) <= 1e-3 * np.abs(d["values"]) + 1e-5).all(), rel.max()
    y16 = crt.forward(x, layer, QuantSpec(bits_a), out="bf16").float().cpu().numpy()
    assert (np.abs(y16 - y32) <= 2.0 ** -8 * np.abs(y32) + 1e-30).all()


# ---------------------------------------------------------------------------
# K1 at larger shapes against the C oracle
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n0", [4, 16, 64, 256])
@pytest.mark.parametrize("family", ["gaussian", "colwise", "rowwise"])
@pytest.mark.parametrize("shape", [(96, 3072), (40, 12288), (33, 1024)])
def test_k1_bit_exact_vs_oracle(n0, family, shape):
    M, K = shape
    xb = O.synth_input(M, K, family, 1000 + n0 + M)
    x = bf16_tensor(xb)
    codes, s32, s64 = crt.rotate_quantize(x, RotationSpec(RotationKind.regular, n0),
                                          QuantSpec(4), scales64=True)
    xd = O.from_bf16_bits(xb)
    rot = O.group_rotate(xd, O.ROT_REGULAR, n0)
    sc = O.compute_scales(rot)
    want = O.pack_int4_rows(O.quantize(rot, sc))
    got = codes[:, :K // 2].cpu().numpy()
    bad = np.argwhere(got != want)
    assert bad.size == 0, (bad[:5], got[tuple(bad[0])], want[tuple(bad[0])])
    assert np.array_equal(s64.cpu().numpy(), sc)


@pytest.mark.parametrize("n0", [16, 256])
def test_k1_f32_input_and_bits8(n0):
    M, K = 64, 3072
    xd = O.synth_outliers(M, K, O.MODE_COLWISE, 50.0, 0.01, 77).astype(np.float32).astype(np.float64)
    x = torch.from_numpy(xd.astype(np.float32)).to(DEV)
    rot = O.group_rotate(xd, O.ROT_REGULAR, n0)
    for bits in (4, 8):
        codes, s32, s64 = crt.rotate_quantize(x, RotationSpec(RotationKind.regular, n0),
                                              QuantSpec(bits), scales64=True)
        sc = O.compute_scales(rot, bits)
        q = O.quantize(rot, sc, bits)
        want = O.pack_int4_rows(q) if bits == 4 else q.view(np.uint8)
        row = crt.packed_row_bytes(K, bits)
        assert np.array_equal(codes[:, :row].cpu().numpy(), want)
        assert np.array_equal(s64.cpu().numpy(), sc)


def test_k1_edge_rows():
    K = 1024
    x = np.zeros((8, K))
    x[1] = 3.5
    x[2, ::2] = 1.0
    x[3] = np.arange(K) - 512.0
    x[4, 5] = -7.0
    x[5] = 1e-38          # subnormal-adjacent tiny values
    x[6] = 3.0e38         # fp32 overflow in the butterflies -> exact row path
    x[7, :8] = [1, -1, 0.5, -0.5, 0.25, 0.125, 2, 4]
    xb = O.to_bf16_bits(x)
    xt = bf16_tensor(xb)
    xd = O.from_bf16_bits(xb)
    for n0 in (4, 16, 64, 256):
        codes, s32, s64 = crt.rotate_quantize(xt, RotationSpec(RotationKind.regular, n0),
                                              QuantSpec(4), scales64=True)
        rot = O.group_rotate(xd, O.ROT_REGULAR, n0)
        sc = O.compute_scales(rot)
        assert np.array_equal(codes[:, :K // 2].cpu().numpy(), O.pack_int4_rows(O.quantize(rot, sc)))
        assert np.array_equal(s64.cpu().numpy(), sc)


@pytest.mark.parametrize("K", [3072, 12288])
@pytest.mark.parametrize("n0", [4, 16])
def test_k1_row_max_settlement_paths(K, n0):
    """The row-max settlement of the rolled kernel: the certified best-chunk
    shortcut (companions within the exponent span), its fallbacks (span too
    wide, subnormal companions, the max tied across chunks / lanes) and
    wide-range rows, in packed and int8-code mode, bit-exact vs the oracle."""
    rng = np.random.default_rng(K + n0)
    M = 48
    x = rng.standard_normal((M, K))
    for r in range(M):
        j = int(rng.integers(0, K // 16)) * 16
        kind = r % 8
        if kind == 0:    # spike, companions in span -> certified shortcut
            x[r, j:j + 16] = 2.0 ** -2
            x[r, j + 3] = 40.0
        elif kind == 1:  # spike, companions far below -> span fails -> exact path
            x[r, j:j + 16] = 2.0 ** -12
            x[r, j + 5] = -40.0
        elif kind == 2:  # subnormal-range companion in the spike's chunk
            x[r, j + 1] = 1e-39
            x[r, j + 7] = 50.0
        elif kind == 3:  # the same spike in two chunks (candidates in both)
            x[r, j + 2] = 45.0
            x[r, (j + 16 * 37) % K + 2] = -45.0
        elif kind == 4:  # wide dynamic range everywhere
            x[r] *= 2.0 ** rng.integers(-20, 20, K)
        elif kind == 5:  # zero chunk next to the maximum
            x[r, j:j + 16] = 0.0
            x[r, (j + 16) % K] = 60.0
    xb = O.to_bf16_bits(x)
    xt = bf16_tensor(xb)
    xd = O.from_bf16_bits(xb)
    spec = RotationSpec(RotationKind.regular, n0)
    rot = O.group_rotate(xd, O.ROT_REGULAR, n0)
    sc = O.compute_scales(rot)
    q = O.quantize(rot, sc)
    codes, s32, s64 = crt.rotate_quantize(xt, spec, QuantSpec(4), scales64=True)
    assert np.array_equal(codes[:, :K // 2].cpu().numpy(), O.pack_int4_rows(q))
    assert np.array_equal(s64.cpu().numpy(), sc)
    c8, s8, sums = crt.rotate_quantize_i8(xt, spec)
    assert np.array_equal(c8[:, :K].cpu().numpy().view(np.int8), q.astype(np.int8))
    assert np.array_equal(s8.cpu().numpy(), sc.astype(np.float32))
    assert np.array_equal(sums.cpu().numpy(), q.astype(np.int64).sum(1))


def test_k1_nonfinite_raises_invalid_value():
    x = torch.randn(4, 256, device=DEV).to(torch.bfloat16)
    x[2, 17] = float("nan")
    with pytest.raises(crt.InvalidValueError):
        crt.rotate_quantize(x, RotationSpec(RotationKind.regular, 16))
    x[2, 17] = float("inf")
    with pytest.raises(crt.InvalidValueError):
        crt.rotate_quantize(x, RotationSpec(RotationKind.regular, 16))
    # the error word was reset: a clean call succeeds afterwards
    crt.rotate_quantize(torch.randn(4, 256, device=DEV).to(torch.bfloat16),
                        RotationSpec(RotationKind.regular, 16))


@pytest.mark.parametrize("n0", [16, 64, 256])
def test_k1_team_slow_rows(n0):
    """Rows the fp32 path cannot certify, in the team kernel at K = 3072 (3
    warps; for N0 >= 64 a lane pair shares a radix-4 digit, k1_team.cuh
    rotate_team): fp32-overflowing groups settled element by element with the
    reference's double arithmetic (group_rotate pipeline.cpp:111-151,
    compute_scales / quantize quant.cpp:10-52), and a NaN in the last warp's
    chunks raising InvalidValueError (quant.cpp:16-18)."""
    M, K = 6, 3072
    x = O.from_bf16_bits(O.synth_input(M, K, "gaussian", 11)).copy()
    x[1, :] = 1.5 * 2.0 ** 126              # every group overflows fp32
    x[3, 2048 + 16:2048 + 80] = -1.25 * 2.0 ** 125  # one block in warp 2
    x[4, 5] = 1.5 * 2.0 ** 126               # a single huge element
    xb = O.to_bf16_bits(x)
    xv = O.from_bf16_bits(xb)
    spec = RotationSpec(RotationKind.regular, n0)
    rot = O.group_rotate(xv, int(spec.kind), n0)
    sc = O.compute_scales(rot)
    q = O.quantize(rot, sc)
    xt = bf16_tensor(xb)
    codes, s32, s64 = crt.rotate_quantize(xt, spec, QuantSpec(4), scales64=True)
    assert np.array_equal(codes[:, :K // 2].cpu().numpy(), O.pack_int4_rows(q))
    assert np.array_equal(s64.cpu().numpy(), sc)
    c8, s8, sums = crt.rotate_quantize_i8(xt, spec)
    assert np.array_equal(c8[:, :K].cpu().numpy().view(np.int8), q.astype(np.int8))
    assert np.array_equal(sums.cpu().numpy(), q.astype(np.int64).sum(1))
    xn = xt.clone()
    xn[2, 2048 + 700] = float("nan")
    with pytest.raises(crt.InvalidValueError):
        crt.rotate_quantize(xn, spec)


@pytest.mark.parametrize("spec", [
    RotationSpec(RotationKind.regular, 0),            # global group (K=1024)
    RotationSpec(RotationKind.sylvester, 32),
    RotationSpec(RotationKind.regular, 16, 0, True),  # identity tail
    RotationSpec(RotationKind.none, 0),
])
def test_k1_exact_kernel_paths(spec):
    M, K = 12, 1024 if spec.identity_tail is False else 1000
    xb = O.synth_input(M, K, "gaussian", 5)
    x = bf16_tensor(xb)
    codes, s32, s64 = crt.rotate_quantize(x, spec, QuantSpec(4), scales64=True)
    rot = O.group_rotate(O.from_bf16_bits(xb), int(spec.kind), spec.group_size, spec.identity_tail)
    sc = O.compute_scales(rot)
    row = crt.packed_row_bytes(K, 4)
    assert np.array_equal(codes[:, :row].cpu().numpy(), O.pack_int4_rows(O.quantize(rot, sc)))
    assert np.array_equal(s64.cpu().numpy(), sc)


# ---------------------------------------------------------------------------
# K3 at FLUX shapes: int32 accumulators bit-exact (row-sampled oracle)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("M,K,N,n0", [(4096, 3072, 3072, 16), (4608, 3072, 12288, 16),
                                      (4608, 12288, 3072, 16), (300, 3072, 640, 256),
                                      (128, 256, 256, 4)])
def test_k3_accumulators_exact_vs_oracle(M, K, N, n0):
    spec = RotationSpec(RotationKind.regular, n0)
    g = torch.Generator().manual_seed(M + K + N)
    x = torch.randn(M, K, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(N, K, generator=g).to(torch.bfloat16).to(DEV)
    bias = torch.randn(N, generator=g).to(DEV)
    layer = crt.prepare_layer(w, bias, spec, QuantSpec(4))
    acc = crt.forward(x, layer, QuantSpec(4), out="i32")
    y32 = crt.forward(x, layer, QuantSpec(4), out="f32")
    codes, sa, sa64 = crt.rotate_quantize(x, spec, QuantSpec(4), scales64=True)
    wc, ws32, ws64 = layer.export()
    rows = np.unique(np.concatenate([np.arange(0, M, max(1, M // 48)), [M - 1]]))
    a_codes = O.unpack_int4_rows_np(codes.cpu().numpy()[rows, :K // 2], K)
    w_codes = O.unpack_int4_rows_np(wc.cpu().numpy(), K)
    want = O.int_gemm(a_codes, w_codes)
    got = acc.cpu().numpy()[rows]
    assert np.array_equal(got, want)
    check_dequant(y32.cpu().numpy()[rows], want, sa64.cpu().numpy()[rows], ws64.cpu().numpy(),
                  bias.cpu().numpy().astype(np.float64))


def test_k3_tails_and_generic_path():
    # M, N not multiples of the 128 x 256 tile; K = 96 takes the CUDA-core path
    for (M, K, N) in [(130, 512, 300), (7, 96, 9), (1, 3072, 18432 // 8)]:
        xb = O.synth_input(M, K, "gaussian", M + N)
        wb = O.synth_input(N, K, "gaussian", M + N + 1)
        x, w = bf16_tensor(xb), bf16_tensor(wb)
        spec = RotationSpec(RotationKind.regular, 16)
        layer = crt.prepare_layer(w, None, spec, QuantSpec(4))
        acc = crt.forward(x, layer, QuantSpec(4), out="i32").cpu().numpy()
        wc, ws = O.prepare_layer(O.from_bf16_bits(wb), O.ROT_REGULAR, 16)
        f = O.forward(O.from_bf16_bits(xb), wc, ws, None, O.ROT_REGULAR, 16)
        assert np.array_equal(acc, f["acc"])


def test_forward_shape_and_bits_errors():
    w = torch.randn(8, 64, device=DEV).to(torch.bfloat16)
    layer = crt.prepare_layer(w, None, RotationSpec(RotationKind.regular, 16))
    with pytest.raises(crt.ShapeError):
        crt.forward(torch.randn(2, 48, device=DEV).to(torch.bfloat16), layer)
    with pytest.raises(crt.InvalidValueError):
        crt.forward(torch.randn(2, 64, device=DEV).to(torch.bfloat16), layer, QuantSpec(5))
    with pytest.raises(crt.ShapeError):
        crt.prepare_layer(w, torch.zeros(3, device=DEV), RotationSpec(RotationKind.regular, 16))


def test_launch_counter_moves():
    before = crt.launch_count()
    crt.rotate_quantize(torch.randn(4, 256, device=DEV).to(torch.bfloat16),
                        RotationSpec(RotationKind.regular, 16))
    assert crt.launch_count() > before


# ---------------------------------------------------------------------------
# Full-size forward, row-sampled oracle: scales are per token,
# so the reference's forward on a row subset X[S, :] is exactly rows S of the
# full result.  The oracle prepares the FULL weights itself; the GPU runs the
# full-size forward (the production path: K1 int8 codes + K3 v3).
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("M,K,N,n0,family", [
    (4096, 3072, 3072, 16, "colwise"),     # configs[0] attn-proj
    (4608, 3072, 12288, 16, "gaussian"),   # configs[1] fc1
    (4608, 12288, 3072, 16, "rowwise"),    # configs[1] fc2
    (4608, 15360, 3072, 16, "colwise"),    # configs[3] single-block proj_out
    (4608, 3072, 3072, 256, "colwise"),    # configs[2] N0 sweep, largest group
])
def test_forward_full_size_row_sampled_vs_oracle(M, K, N, n0, family):
    xb = O.synth_input(M, K, family, 41)
    wb = O.synth_input(N, K, "gaussian", 42)
    bias = O.from_bf16_bits(O.to_bf16_bits(O.gaussian_matrix(1, N, 43)[0]))
    spec = RotationSpec(RotationKind.regular, n0)
    layer = crt.prepare_layer(bf16_tensor(wb), torch.from_numpy(bias).float().to(DEV), spec)
    x = bf16_tensor(xb)
    acc = crt.forward(x, layer, QuantSpec(4), out="i32").cpu().numpy()
    y32 = crt.forward(x, layer, QuantSpec(4), out="f32").cpu().numpy().astype(np.float64)
    rows = np.unique(np.concatenate([np.linspace(0, M - 1, 40).astype(np.int64), [1, M - 2]]))
    wc, ws = O.prepare_layer(O.from_bf16_bits(wb), O.ROT_REGULAR, n0)
    f = O.forward(O.from_bf16_bits(xb[rows]), wc, ws, bias, O.ROT_REGULAR, n0)
    assert np.array_equal(acc[rows], f["acc"])
    want = f["values"]
    assert (np.abs(y32[rows] - want) <= 1e-6 * np.abs(want) + 1e-6).all()
