"""K3 v3 (hardware-expanded weights) accumulators / dequant vs an integer
reference built from the exported codes (dev aid)."""
import sys
import time
sys.path.insert(0, ".")
import torch
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec

def unpack(c, k):
    c = c[:, : k // 2].to(torch.int32)
    lo, hi = c & 0xF, (c >> 4) & 0xF
    lo = torch.where(lo >= 8, lo - 16, lo)
    hi = torch.where(hi >= 8, hi - 16, hi)
    return torch.stack([lo, hi], dim=2).reshape(c.shape[0], k)

for (M, K, N) in [(256, 128, 256), (384, 3072, 768), (4096, 3072, 3072), (4608, 12288, 3072), (4608, 3072, 12288)]:
    torch.manual_seed(0)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    spec = RotationSpec(RotationKind.regular, 16)
    layer = crt.prepare_layer(w, torch.randn(N, device="cuda"), spec)
    codes_p, sa = crt.rotate_quantize(x, spec)
    codes8, sa8, sums = crt.rotate_quantize_i8(x, spec)
    A = unpack(codes_p, K)
    a8 = codes8[:, :K].view(torch.int8).to(torch.int32)
    ok_codes = torch.equal(A, a8) and torch.equal(sa, sa8) and torch.equal(A.sum(1), sums)
    wc = layer.export(scales64=False)[0]
    B = unpack(wc, K)
    ref = (A.double() @ B.double().T).round().to(torch.int64)
    acc = crt.quant_gemm_i8(codes8, sa8, sums, layer, out="i32").to(torch.int64)
    torch.cuda.synchronize()
    bad = int((acc != ref).sum())
    y2 = crt.quant_gemm(codes_p, sa, layer, out="f32")
    y3 = crt.quant_gemm_i8(codes8, sa8, sums, layer, out="f32")
    yb2 = crt.quant_gemm(codes_p, sa, layer, out="bf16")
    yb3 = crt.quant_gemm_i8(codes8, sa8, sums, layer, out="bf16")
    torch.cuda.synchronize()
    print(f"M={M} K={K} N={N}: codes_i8_ok={ok_codes} acc_mismatch={bad} f32_equal_v2={torch.equal(y2, y3)} bf16_equal_v2={torch.equal(yb2, yb3)}", flush=True)
    if bad:
        idx = (acc != ref).nonzero()
        r, c = int(idx[0, 0]), int(idx[0, 1])
        print("   first", r, c, int(acc[r, c]), int(ref[r, c]), "rows", torch.unique(idx[:,0]).numel(), "cols", torch.unique(idx[:,1]).numel())
    # timing
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        crt.quant_gemm_i8(codes8, sa8, sums, layer, y=yb)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        crt.quant_gemm_i8(codes8, sa8, sums, layer, y=yb)
    e.record(); e.synchronize()
    t = s.elapsed_time(e) / 10 * 1e3
    print(f"   v3 {t:.1f} us  {2*M*N*K/t/1e6:.0f} TOPS", flush=True)
