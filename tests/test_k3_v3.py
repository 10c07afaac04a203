"""The int8-activation-code K3 (v4 by default: packed weights expanded by
expander warps into tensor memory; v3 with CRT_K3_V3=1, re-run by
tests/test_alt_paths.py: tcgen05.cp decompression) against the exact
integer GEMM of the same codes and against the packed v2 path.  The int_gemm accumulators must be bit-exact
(pipeline.cpp:178-204) and the dequantised outputs identical to v2's, which
tests/test_gpu_parity.py pins to the oracle.  Shapes cover ragged token tiles
(M not a multiple of 192), ragged channel tiles (N not a multiple of 256),
partial 128-code K blocks (K % 128 != 0, K % 32 != 0) and the FLUX shapes."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _unpack(c, k):
    c = c[:, : (k + 1) // 2].to(torch.int32)
    lo, hi = c & 0xF, (c >> 4) & 0xF
    lo = torch.where(lo >= 8, lo - 16, lo)
    hi = torch.where(hi >= 8, hi - 16, hi)
    return torch.stack([lo, hi], dim=2).reshape(c.shape[0], -1)[:, :k]


SHAPES = [(1, 32, 16), (5, 96, 40), (7, 40, 24), (65, 100, 300), (193, 160, 257),
          (384, 3072, 768), (257, 3104, 1000), (1024, 12288, 512), (4096, 3072, 3072),
          # few tokens (FLUX AdaLN: M = 1, N = 18432)
          (1, 3072, 18432), (8, 3072, 9216), (3, 12288, 3072), (2, 3104, 700), (8, 48, 33)]


@pytest.mark.parametrize("M,K,N", SHAPES)
@pytest.mark.parametrize("n0", [4, 16])
def test_v3_accumulators_exact(M, K, N, n0):
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import RotationKind, RotationSpec
    if K % n0:
        pytest.skip("K not a multiple of the rotation group")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + K + N)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    x[0, :: max(1, K // 5)] *= 40  # outlier columns
    w = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    spec = RotationSpec(RotationKind.regular, n0)
    layer = crt.prepare_layer(w, torch.randn(N, device="cuda", generator=g), spec)
    codes_p, sa = crt.rotate_quantize(x, spec)
    codes8, sa8, sums = crt.rotate_quantize_i8(x, spec)
    A = _unpack(codes_p, K)
    a8 = codes8[:, :K].view(torch.int8).to(torch.int32)
    assert torch.equal(A, a8), "int8 codes differ from the packed codes"
    assert torch.equal(sa, sa8)
    assert torch.equal(A.sum(1), sums)
    B = _unpack(layer.export(scales64=False)[0], K)
    ref = (A.double() @ B.double().T).round().to(torch.int64)
    acc = crt.quant_gemm_i8(codes8, sa8, sums, layer, out="i32").to(torch.int64)
    assert torch.equal(acc, ref)
    for out in ("f32", "bf16"):
        y2 = crt.quant_gemm(codes_p, sa, layer, out=out)
        y3 = crt.quant_gemm_i8(codes8, sa8, sums, layer, out=out)
        assert torch.equal(y2, y3), out


@pytest.mark.parametrize("M,K,N", [(8, 64, 16), (193, 160, 257), (33, 48, 70), (4608, 3072, 12288)])
def test_forward_v3_equals_packed_path(M, K, N):
    """crt_forward routes W4A4 through K1 bits-5 + v3; its
    output must equal K1 bits-4 + the packed GEMM."""
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import RotationKind, RotationSpec
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    spec = RotationSpec(RotationKind.regular, 16)
    layer = crt.prepare_layer(w, torch.randn(N, device="cuda", generator=g), spec)
    codes_p, sa = crt.rotate_quantize(x, spec)
    for out in ("i32", "f32", "bf16"):
        assert torch.equal(crt.forward(x, layer, out=out), crt.quant_gemm(codes_p, sa, layer, out=out))


@pytest.mark.parametrize("M,K,N", [(1, 16, 16), (7, 48, 40), (193, 160, 257), (384, 3072, 768),
                                   (257, 3104, 1000), (1024, 12288, 512)])
def test_v3_w8a8_accumulators_exact(M, K, N):
    """f1: W8A8 on the v3 kernel (int8 weights copied to TMEM
    by tcgen05.cp without decompression).  int_gemm exact; the dequantised
    outputs equal crt_dequant of the same accumulators (one fp32 expression)."""
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec
    g = torch.Generator(device="cuda").manual_seed(M + 3 * K + N)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    spec, q8 = RotationSpec(RotationKind.regular, 16), QuantSpec(8)
    layer = crt.prepare_layer(w, torch.randn(N, device="cuda", generator=g), spec, q8)
    codes, sa = crt.rotate_quantize(x, spec, q8)
    A = codes[:, :K].view(torch.int8).to(torch.float64)
    B = layer.export(scales64=False)[0][:, :K].view(torch.int8).to(torch.float64)
    ref = (A @ B.T).round().to(torch.int64)
    acc = crt.quant_gemm(codes, sa, layer, q8, out="i32")
    assert torch.equal(acc.to(torch.int64), ref)
    for out in ("f32", "bf16"):
        assert torch.equal(crt.quant_gemm(codes, sa, layer, q8, out=out),
                           crt.dequant(acc, sa, layer, out=out)), out
    assert torch.equal(crt.forward(x, layer, q8, out="i32"), acc)


@pytest.mark.parametrize("M,K,N,ldy", [(300, 3072, 1000, 1024), (257, 3104, 700, 712), (5, 3072, 300, 320),
                                       (193, 1536, 40, 48)])
@pytest.mark.parametrize("out", ["bf16", "f32"])
def test_forward_into_wider_rows(M, K, N, ldy, out):
    """y as a column block of a wider row-major buffer (ldy > N): the K3
    epilogue (v4's TMA-store boxes clip at N through the tensor map; the GEMV
    and the per-lane stores index with ldy) must write exactly the [M, N]
    block, leave the columns beyond N untouched, and equal the contiguous
    forward."""
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import RotationKind, RotationSpec
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(M + N)
    x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(N, K, device=dev, generator=g).to(torch.bfloat16)
    b = torch.randn(N, device=dev, generator=g)
    layer = crt.prepare_layer(w, b, RotationSpec(RotationKind.regular, 16))
    ref = crt.forward(x, layer, out=out)
    dt = torch.bfloat16 if out == "bf16" else torch.float32
    big = torch.full((M, ldy), 7.0, dtype=dt, device=dev)
    crt.forward(x, layer, out=out, y=big[:, :N])
    torch.cuda.synchronize()
    assert torch.equal(big[:, :N], ref)
    assert bool((big[:, N:] == 7.0).all())
